// Per-rank B200 execution context (see gpu_context.hpp for the reference map).
#include "foundry/gpu_context.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>

#include <cuda_runtime.h>

namespace foundry {

namespace {
// FOUNDRY_DEBUG driver-call accounting: total ns and calls per kind
enum StatKind { kGetFunction, kFuncLoad, kSetAttribute, kLibraryLoad, kGetKernel, kStatKinds };
std::atomic<uint64_t> g_stat_ns[kStatKinds], g_stat_n[kStatKinds];
struct StatScope {
    StatKind k;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit StatScope(StatKind kind) : k(kind) {}
    ~StatScope() {
        g_stat_ns[k] += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
        g_stat_n[k] += 1;
    }
};
uint64_t align_down(uint64_t v, uint64_t a) { return v / a * a; }
uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }
std::string key_of(uint64_t hash, std::string_view name) { return hex16(hash) + "|" + std::string(name); }
}  // namespace

GpuContext::GpuContext(Device& dev) : dev_(dev) {
    const DriverApi& api = driver();
    dev_.make_current();
    CUdevice d = 0;
    cu_check(api.cuCtxGetDevice(&d), "cuCtxGetDevice");
    cu_device_ = d;
}

GpuContext::~GpuContext() {
    const DriverApi* api = nullptr;
    try {
        api = &driver();
    } catch (...) {
        return;
    }
    cudaSetDevice(dev_.ordinal());
    cudaDeviceSynchronize();
    for (auto& l : libs_)
        if (l.lib) api->cuLibraryUnload(l.lib);
    if (phys_at_ && phys_bytes_) api->cuMemUnmap(phys_at_, phys_bytes_);
    if (phys_) api->cuMemRelease(phys_);
    if (va_) api->cuMemAddressFree(va_, va_bytes_);
}

std::string driver_call_stats(bool reset) {
    static const char* names[kStatKinds] = {"cuKernelGetFunction", "cuFuncLoad", "cuFuncSetAttribute",
                                            "cuLibraryLoadData", "cuLibraryGet*"};
    std::string out;
    char line[160];
    for (int k = 0; k < kStatKinds; ++k) {
        const uint64_t n = reset ? g_stat_n[k].exchange(0) : g_stat_n[k].load();
        const uint64_t ns = reset ? g_stat_ns[k].exchange(0) : g_stat_ns[k].load();
        std::snprintf(line, sizeof line, "%s %llu calls %.3f ms (%.2f us each); ", names[k], (unsigned long long)n,
                      ns * 1e-6, n ? ns * 1e-3 / n : 0.0);
        out += line;
    }
    return out;
}

// ------------------------------------------------------------------ libraries

GpuContext::OpenedLibrary GpuContext::open_library(const KernelImage& image,
                                                   std::span<const uint8_t> cubin) const {
    const DriverApi& api = driver();
    dev_.make_current();
    OpenedLibrary o;
    {
        StatScope st(kLibraryLoad);
        cu_check(api.cuLibraryLoadData(&o.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0),
                 "cuLibraryLoadData");
    }
    StatScope st(kGetKernel);
    try {
        size_t sz = 0;
        cu_check(api.cuLibraryGetGlobal(&o.ctx_global, &sz, o.lib, "fdy_trace_context"),
                 "cuLibraryGetGlobal(fdy_trace_context)");
        cu_check(api.cuLibraryGetGlobal(&o.init_global, &sz, o.lib, "fdy_device_inited"),
                 "cuLibraryGetGlobal(fdy_device_inited)");
        o.kernels.resize(image.entrypoints.size());
        for (size_t i = 0; i < image.entrypoints.size(); ++i)
            cu_check(api.cuLibraryGetKernel(&o.kernels[i], o.lib, image.entrypoints[i].name.c_str()),
                     "cuLibraryGetKernel");
    } catch (...) {
        api.cuLibraryUnload(o.lib);
        throw;
    }
    return o;
}

uint32_t GpuContext::load_library(uint64_t hash, const KernelImage& image,
                                  std::span<const uint8_t> cubin, uint32_t ordinal,
                                  bool requires_init) {
    return register_library(hash, image, open_library(image, cubin), ordinal, requires_init);
}

CUfunction GpuContext::function(const Kernel& k) const {
    std::lock_guard lock(fn_mu_);
    if (!k.fn) {
        dev_.make_current();
        StatScope st(kGetFunction);
        cu_check(driver().cuKernelGetFunction(&k.fn, k.kern), "cuKernelGetFunction");
    }
    return k.fn;
}

void GpuContext::ensure_loaded(const Kernel& k) const {
    const CUfunction f = function(k);
    std::lock_guard lock(fn_mu_);
    if (k.loaded) return;
    StatScope st(kFuncLoad);
    if (driver().cuFuncLoad) cu_check(driver().cuFuncLoad(f), "cuFuncLoad");
    k.loaded = true;
}

// Launch limits go on the kernel's function in THIS context
// (cuFuncSetAttribute, ~0.1 us) rather than on the context-independent
// CUkernel (cuKernelSetAttribute, 10-40 us and serialized in the driver:
// 5358 calls cost 50-200 ms of LOAD on the headline set; tools/gpu_restore_study.sh).
// Graph nodes and launches use that function, so the limit applies to them.
void GpuContext::set_kernel_attribute(const Kernel& k, CUfunction_attribute attr, int value) const {
    const CUfunction f = function(k);
    StatScope st(kSetAttribute);
    cu_check(driver().cuFuncSetAttribute(f, attr, value), "cuFuncSetAttribute");
}

void GpuContext::require_dynamic_smem(const Kernel& k, int bytes) const {
    {
        std::lock_guard lock(fn_mu_);
        if (bytes <= k.max_dynamic_smem) return;
    }
    set_kernel_attribute(k, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, bytes);
    std::lock_guard lock(fn_mu_);
    k.max_dynamic_smem = std::max(k.max_dynamic_smem, bytes);
}

void GpuContext::set_carveout(const Kernel& k, int percent) const {
    {
        std::lock_guard lock(fn_mu_);
        if (percent == k.carveout) return;
    }
    set_kernel_attribute(k, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, percent);
    std::lock_guard lock(fn_mu_);
    k.carveout = percent;
}

int GpuContext::function_attribute(const Kernel& k, CUfunction_attribute attr) const {
    int v = 0;
    cu_check(driver().cuFuncGetAttribute(&v, attr, function(k)), "cuFuncGetAttribute");
    return v;
}

uint32_t GpuContext::register_library(uint64_t hash, const KernelImage& image, OpenedLibrary&& o,
                                      uint32_t ordinal, bool requires_init) {
    Library L;
    L.hash = hash;
    L.requires_init = requires_init;
    L.lib = o.lib;
    L.ctx_global = o.ctx_global;
    L.init_global = o.init_global;
    o.lib = nullptr;
    const uint32_t li = static_cast<uint32_t>(libs_.size());
    libs_.push_back(L);
    for (uint32_t i = 0; i < image.entrypoints.size(); ++i) {
        const KernelEntry& e = image.entrypoints[i];
        Kernel k;
        k.kern = o.kernels[i];
        k.library = li;
        k.entry_index = i;
        k.entry_id = (ordinal << 16) | i;
        k.arg_buffer_size = e.arg_buffer_size;
        k.hidden_offsets = e.hidden_offsets;
        k.attrs = e.attrs;
        k.name = e.name;
        k.binary_hash = hash;
        const uint32_t ki = static_cast<uint32_t>(kernels_.size());
        kernel_index_[key_of(hash, e.name)] = ki;
        by_entry_id_[k.entry_id] = ki;
        kernels_.push_back(std::move(k));
    }
    c_module_load.fetch_add(1);
    return li;
}

void GpuContext::run_device_init(uint32_t library) {
    require(library < libs_.size(), Errc::invalid_argument, "unknown module handle");
    Library& L = libs_[library];
    require(L.requires_init, Errc::invalid_argument, "module does not require device-side init");
    const uint32_t one = 1;
    dev_.make_current();
    cuda_check(cudaMemcpy(reinterpret_cast<void*>(L.init_global), &one, 4, cudaMemcpyHostToDevice),
               "device-side init");
    L.inited = true;
    c_device_init.fetch_add(1);
}

bool GpuContext::library_device_inited(uint32_t l) const { return libs_.at(l).inited; }
bool GpuContext::library_requires_init(uint32_t l) const { return libs_.at(l).requires_init; }

const GpuContext::Kernel* GpuContext::find_kernel(uint64_t hash, std::string_view name) const {
    auto it = kernel_index_.find(key_of(hash, name));
    return it == kernel_index_.end() ? nullptr : &kernels_[it->second];
}

const GpuContext::Kernel* GpuContext::kernel_by_entry_id(uint32_t id) const {
    auto it = by_entry_id_.find(id);
    return it == by_entry_id_.end() ? nullptr : &kernels_[it->second];
}

const GpuContext::Kernel* GpuContext::kernel_by_handle(CUfunction fn, CUkernel kern) const {
    std::lock_guard lock(fn_mu_);  // fn is filled lazily under this lock
    for (const auto& k : kernels_)
        if ((fn && k.fn == fn) || (kern && k.kern == kern)) return &k;
    if (fn) {  // a function handle obtained outside function(): compare through the kernel
        for (const auto& k : kernels_) {
            CUfunction f = nullptr;
            if (driver().cuKernelGetFunction(&f, k.kern) == CUDA_SUCCESS && f == fn) {
                k.fn = f;
                return &k;
            }
        }
    }
    return nullptr;
}

bool GpuContext::has_library(uint64_t hash) const {
    for (const auto& l : libs_)
        if (l.hash == hash) return true;
    return false;
}

// ------------------------------------------------------------------ region

void GpuContext::reserve_region(const RegionConfig& cfg, uint64_t backed_bytes, bool allow_relocation) {
    require(cfg.capacity > 0, Errc::invalid_argument, "zero capacity region");
    require(cfg.granularity > 0 && (cfg.granularity & (cfg.granularity - 1)) == 0,
            Errc::invalid_argument, "granularity must be a power of two");
    require(cfg.capacity % cfg.granularity == 0, Errc::invalid_argument,
            "capacity must be a multiple of the granularity");
    require(!reserved_, Errc::invalid_argument, "region already reserved");
    const DriverApi& api = driver();
    dev_.make_current();
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = dev_.ordinal();
    size_t gran = 0;
    cu_check(api.cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM),
             "cuMemGetAllocationGranularity");
    gran = std::max<size_t>(gran, cfg.granularity);

    captured_base_ = cfg.base;
    logical_ = cfg;
    const uint64_t lo = align_down(cfg.base, gran);
    va_bytes_ = align_up(cfg.base + cfg.capacity, gran) - lo;
    cu_check(api.cuMemAddressReserve(&va_, va_bytes_, gran, lo, 0), "cuMemAddressReserve");
    if (va_ != lo) {
        if (!allow_relocation) {
            const uint64_t got = va_;
            api.cuMemAddressFree(va_, va_bytes_);
            va_ = 0;
            raise(Errc::out_of_region,
                  "cannot reserve the captured VA range at 0x" + hex16(cfg.base) +
                      " (the driver placed it at 0x" + hex16(got) + "); load with relocation enabled");
        }
        logical_.base = va_;  // relocate: K1 rebases embedded addresses onto va_
    }
    // physical backing for [va_, base + backed_bytes); grows on demand
    phys_bytes_ = align_up(std::max<uint64_t>(logical_.base - va_ + backed_bytes, 1), gran);
    cu_check(api.cuMemCreate(&phys_, phys_bytes_, &prop, 0), "cuMemCreate");
    cu_check(api.cuMemMap(va_, phys_bytes_, 0, phys_, 0), "cuMemMap");
    phys_at_ = va_;
    CUmemAccessDesc acc{};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    cu_check(api.cuMemSetAccess(va_, phys_bytes_, &acc, 1), "cuMemSetAccess");
    bitmap_.assign((cfg.capacity / cfg.granularity + 63) / 64, 0);
    reserved_ = true;
    c_reserve.fetch_add(1);
}

void GpuContext::mark(uint64_t addr, uint64_t len, bool on) {
    const uint64_t g0 = (addr - logical_.base) / logical_.granularity;
    const uint64_t g1 = (addr + len - logical_.base + logical_.granularity - 1) / logical_.granularity;
    for (uint64_t g = g0; g < g1 && g / 64 < bitmap_.size(); ++g) {
        if (on) bitmap_[g / 64] |= 1ull << (g % 64);
        else bitmap_[g / 64] &= ~(1ull << (g % 64));
    }
    bitmap_dirty_ = true;
}

bool GpuContext::address_mapped(uint64_t a) const {
    if (!reserved_ || a < logical_.base) return false;
    const uint64_t g = (a - logical_.base) / logical_.granularity;
    if (g / 64 >= bitmap_.size()) return false;
    return (bitmap_[g / 64] >> (g % 64)) & 1ull;
}

uint64_t GpuContext::allocate(uint64_t size) {
    require(reserved_, Errc::invalid_argument, "region not reserved");
    require(size > 0, Errc::invalid_argument, "zero-byte allocation");
    require(size <= logical_.capacity, Errc::out_of_region,
            "allocation of " + std::to_string(size) + " bytes exceeds region capacity");
    const uint64_t len = align_up(size, logical_.granularity);
    const uint64_t limit = prealloc_limit_.value_or(logical_.capacity);
    require(offset_ + len <= limit, Errc::out_of_region,
            "allocation of " + std::to_string(size) + " bytes exceeds " +
                (prealloc_limit_ ? "the preallocated range" : "region capacity"));
    const uint64_t addr = logical_.base + offset_;
    offset_ += len;
    // grow the physical backing if a (non-preallocated) grant runs past it
    if (addr + len > phys_at_ + phys_bytes_)
        raise(Errc::out_of_region, "allocation at 0x" + hex16(addr) +
                                       " runs past the backed range (manifest final offset)");
    if (!prealloc_limit_) {
        mark(addr, len, true);
        c_map.fetch_add(1);
    }
    c_grants.fetch_add(1);
    records_.push_back({records_.size(), size, addr, len,
                        recording_window_ ? AllocWindow::capture_window : AllocWindow::pre_capture});
    live_.emplace_back(addr, len);
    return addr;
}

void GpuContext::free(uint64_t address) {
    auto it = std::find_if(live_.begin(), live_.end(), [&](const auto& g) { return g.first == address; });
    require(it != live_.end(), Errc::unknown_address,
            "free of address 0x" + hex16(address) + " that was never granted");
    mark(it->first, it->second, false);  // the granule leaks; only the mapping goes
    c_unmap.fetch_add(1);
    live_.erase(it);
}

void GpuContext::preallocate(uint64_t final_offset) {
    require(final_offset % logical_.granularity == 0, Errc::invalid_argument,
            "final offset must be granularity-aligned");
    require(final_offset <= logical_.capacity, Errc::out_of_region, "final offset exceeds region capacity");
    require(offset_ == 0 && records_.empty(), Errc::invalid_argument,
            "preallocate must precede all allocations");
    if (final_offset > 0) {
        mark(logical_.base, final_offset, true);
        c_map.fetch_add(1);
    }
    prealloc_limit_ = final_offset;
}

void GpuContext::begin_capture_window() {
    require(!recording_window_, Errc::invalid_argument, "capture window already open");
    recording_window_ = true;
}

void GpuContext::replay_capture_window(const MemoryEventLog& log) {
    require(!recording_window_, Errc::invalid_argument, "cannot replay inside an open window");
    require(offset_ == log.starting_offset, Errc::layout_divergence,
            "region offset 0x" + hex16(offset_) + " does not match the recorded pre-window offset 0x" +
                hex16(log.starting_offset));
    recording_window_ = true;
    try {
        for (const auto& rec : log.records) {
            if (rec.window != AllocWindow::capture_window) continue;
            const uint64_t granted = allocate(rec.size);
            require(granted - logical_.base == rec.address - log.config.base, Errc::layout_divergence,
                    "window replay placed 0x" + hex16(granted) + " where the log expects 0x" +
                        hex16(rec.address));
        }
    } catch (...) {
        recording_window_ = false;
        throw;
    }
    recording_window_ = false;
    require(offset_ == log.final_offset, Errc::layout_divergence,
            "window replay ended at offset 0x" + hex16(offset_) + ", log expects 0x" +
                hex16(log.final_offset));
}

void GpuContext::zero_region() {
    if (!phys_at_) return;
    dev_.make_current();
    cuda_check(cudaMemsetAsync(reinterpret_cast<void*>(phys_at_), 0, phys_bytes_, dev_.stream()),
               "cudaMemsetAsync(region)");
}

// ------------------------------------------------------------------ trace

void GpuContext::ensure_trace_arena(uint64_t bytes) {
    if (trace_arena_.size() >= bytes) return;
    trace_arena_ = DeviceBuffer(dev_, bytes);
    published_.clear();  // ctx contents change; re-upload below
    bitmap_dirty_ = true;
}

void GpuContext::sync_trace_state() {
    dev_.make_current();
    const size_t bm_bytes = bitmap_.size() * 8;
    if (!trace_meta_.data()) {
        trace_meta_ = DeviceBuffer(dev_, 128 + bm_bytes);
        d_ctx_ = reinterpret_cast<fdy_trace_ctx*>(trace_meta_.data());
        d_cursor_ = reinterpret_cast<unsigned long long*>(trace_meta_.data() + 64);
        d_bitmap_ = reinterpret_cast<uint64_t*>(trace_meta_.data() + 128);
        bitmap_dirty_ = true;
        // pool memory is not zeroed: a path that launches before any reset_trace
        // (naive_rebuild_all) must not start from a stale cursor
        cuda_check(cudaMemsetAsync(trace_meta_.data(), 0, 128, dev_.stream()), "trace meta reset");
        cuda_check(cudaStreamSynchronize(dev_.stream()), "trace meta reset");
    }
    if (bitmap_dirty_) {
        fdy_trace_ctx h{};
        h.arena = trace_arena_.data();
        h.cursor = d_cursor_;
        h.capacity = trace_arena_.size();
        h.bitmap = d_bitmap_;
        h.map_base = logical_.base;
        h.map_granules = logical_.capacity / logical_.granularity;
        h.granule_shift = static_cast<uint32_t>(__builtin_ctzll(logical_.granularity));
        cuda_check(cudaMemcpy(d_ctx_, &h, sizeof h, cudaMemcpyHostToDevice), "trace ctx upload");
        if (bm_bytes)
            cuda_check(cudaMemcpy(d_bitmap_, bitmap_.data(), bm_bytes, cudaMemcpyHostToDevice),
                       "mapping bitmap upload");
        bitmap_dirty_ = false;
    }
    for (uint32_t i = static_cast<uint32_t>(published_.size()); i < libs_.size(); ++i) {
        const fdy_trace_ctx* p = d_ctx_;
        cuda_check(cudaMemcpy(reinterpret_cast<void*>(libs_[i].ctx_global), &p, sizeof p,
                              cudaMemcpyHostToDevice),
                   "publish trace ctx");
        published_.push_back(i);
    }
}

void GpuContext::reset_trace() {
    dev_.make_current();
    cuda_check(cudaMemsetAsync(d_cursor_, 0, 8, dev_.stream()), "trace reset");
}

std::vector<uint8_t> GpuContext::read_trace() {
    dev_.make_current();
    unsigned long long used = 0;
    cuda_check(cudaMemcpyAsync(&used, d_cursor_, 8, cudaMemcpyDeviceToHost, dev_.stream()), "trace D2H");
    cuda_check(cudaStreamSynchronize(dev_.stream()), "trace sync");
    used = std::min<unsigned long long>(used, trace_arena_.size());
    std::vector<uint8_t> out(used);
    if (used)
        cuda_check(cudaMemcpy(out.data(), trace_arena_.data(), used, cudaMemcpyDeviceToHost), "trace D2H");
    return out;
}

// ------------------------------------------------------------------ counters

CounterSnapshot GpuContext::counters() const {
    CounterSnapshot s;
    s["alloc.reserve_calls"] = c_reserve.load();
    s["alloc.map_calls"] = c_map.load();
    s["alloc.unmap_calls"] = c_unmap.load();
    s["alloc.grants"] = c_grants.load();
    s["module.load_calls"] = c_module_load.load();
    s["module.device_init_calls"] = c_device_init.load();
    s["capture.begin_calls"] = 0;
    s["capture.launch_calls"] = 0;
    s["capture.node_records"] = 0;
    s["capture.edge_records"] = 0;
    s["graph.add_node_calls"] = c_add_node.load();
    s["graph.add_edge_calls"] = c_add_edge.load();
    s["graph.set_attr_calls"] = c_set_attr.load();
    s["exec.instantiate_calls"] = c_instantiate.load();
    s["exec.update_calls"] = c_update.load();
    s["exec.update_nodes_touched"] = c_update_touched.load();
    s["replay.launch_calls"] = c_replay.load();
    return s;
}

}  // namespace foundry
