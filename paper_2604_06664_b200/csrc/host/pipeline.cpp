// LOAD orchestration on B200 (phase map and reference anchors: pipeline.hpp).
#include "foundry/pipeline.hpp"
#include "foundry/device_pack.hpp"

#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <future>
#include <mutex>
#include <thread>

#include <cuda_runtime.h>

#include "foundry/bytes.hpp"
#include "foundry/capture.hpp"
#include "../kernels/fdy_kernels.h"
#include "foundry/parallel.hpp"
#include "foundry/staging.hpp"
#include "foundry/template_store.hpp"
#include "foundry/trace_module.hpp"
#include "foundry/workload.hpp"

namespace foundry {

namespace fs = std::filesystem;

namespace {

using Clock = std::chrono::steady_clock;

// Driver lane: the reference serializes driver mutation, instantiation and
// update on one lane (sim_driver.hpp:213-215). The CUDA driver does too,
// behind process-wide locks, and concurrent LOADs (or teardowns) from several
// threads of one process convoy on them (profiles/round2_thread_vs_process.md).
// Even with only the driver-bound phases on one lane, another LOAD's staging
// (allocations, copies, CRC launches) stretched a concurrent cuGraphInstantiate
// by up to 15x. So a LOAD and a context's teardown hold one process-wide lane:
// LOADs of one process run one after another (N x one LOAD); parallel LOADs
// are one process per GPU (bench.py, tools/verify_tp8.py).
std::mutex& driver_lane() {
    static std::mutex m;
    return m;
}

double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

constexpr uint32_t kNoMember = 0xFFFFFFFFu;

// FOUNDRY_DEBUG=1 prints LOAD phase boundaries to stderr (diagnostics only),
// in ms since this library's static initialization (~process start for the CLI).
const auto g_debug_t0 = Clock::now();
void debug_phase(const char* what) {
    static const bool on = std::getenv("FOUNDRY_DEBUG") != nullptr;
    if (on) std::fprintf(stderr, "[foundry] %9.3f ms  %s\n", ms_since(g_debug_t0), what);
}
uint64_t rd64(const uint8_t* p) {
    uint64_t v;
    std::memcpy(&v, p, 8);
    return v;
}

}  // namespace

struct ServingContext::Impl {
    std::unique_ptr<Device> owned_dev;
    Device* dev = nullptr;
    fs::path root;
    std::unique_ptr<GpuContext> ctx;
    LoadOptions opts;
    LoadTimings t;
    Manifest manifest;
    Catalog catalog;

    std::unique_ptr<StagedArchive> staged;  // every listed file, in pinned host memory and HBM

    // reference archives without templates.fdt: the GPU packer's host copy
    // (header + host sections; the device-only sections stay in HBM)
    std::unique_ptr<uint8_t[]> inline_store;
    std::span<const uint8_t> store_host;
    std::unique_ptr<StoreView> view;
    DeviceStore dstore;
    DeviceBuffer d_members;  // every member image, materialized in HBM
    // host copies of member images, fetched on first use (the representatives
    // at LOAD; other members when served) — parameters stay resident in HBM
    std::unique_ptr<uint8_t[]> h_members;
    std::vector<uint8_t> h_present;
    mutable std::mutex fetch_mu;
    std::vector<int32_t> kernel_of;  // store kernel index -> GpuContext kernel (or -1)

    struct Group {
        CUgraph graph = nullptr;
        CUgraphExec exec = nullptr;
        std::vector<CUgraphNode> nodes;
        uint32_t applied = kNoMember;  // member index currently in the exec
        uint32_t bound = kNoMember;    // group whose member that is (share_execs: any of the shape)
        // device_updates: per-node device handles + what each node was built with
        std::vector<FdyServeNode> serve_nodes;
        DeviceBuffer d_serve_nodes;
        std::vector<std::array<uint64_t, 3>> memops;  // memop records currently in the exec
        std::vector<uint32_t> memop_nodes;            // node index of memop slot k
        uint32_t n_kernel_nodes = 0;
    };
    // device_updates serve plan (computed once at LOAD by fdy_serve_plan_kernel)
    std::vector<uint8_t> serve_member_host;           // per member: host path needed
    std::vector<uint32_t> serve_memop_base;           // per member: first slot in serve_plan_records
    std::vector<std::array<uint64_t, 3>> serve_plan_records;
    // device updates that failed since the last check (host-mapped; the serve
    // kernel writes them, replay() reads them): u32 "any" word, then one flag
    // byte per member
    PinnedBuffer serve_error;
    void build_serve_plan();
    bool recover_device_serve(uint32_t gi);
    uint64_t serve_on_device(uint32_t gi, uint32_t m);
    std::vector<Group> groups;
    // share_execs: the group whose graph/exec serves group g (itself otherwise)
    std::vector<uint32_t> owner;
    Group& exec_of(uint32_t g) { return groups[owner.empty() ? g : owner[g]]; }
    std::vector<uint32_t> labels;
    uint64_t lane_acquisitions = 0;
    std::mutex stats_mu;
    CUcontext cu_ctx = nullptr;

    ~Impl() {
        std::lock_guard lane(driver_lane());
        try {
            const DriverApi& api = driver();
            if (dev) dev->make_current();
            for (auto& g : groups) {
                if (g.exec) api.cuGraphExecDestroy(g.exec);
                if (g.graph) api.cuGraphDestroy(g.graph);
            }
        } catch (...) {
        }
        ctx.reset();  // libraries, then VA (destroy order: execs -> graphs -> libraries -> VA)
    }

    std::span<const uint8_t> file_host(const std::string& rel) const { return staged->host(rel); }

    // Host view of member m's image; copied out of HBM on first use.
    const uint8_t* member_image(uint32_t m) const {
        const fdt_member& M = view->member(m);
        uint8_t* dst = h_members.get() + M.out_off;
        std::lock_guard lock(fetch_mu);
        if (!h_present[m]) {
            dev->make_current();
            cuda_check(cudaMemcpy(dst, d_members.data() + M.out_off, view->group(M.group).image_bytes,
                                  cudaMemcpyDeviceToHost),
                       "cudaMemcpy(member image D2H)");
            view->check_image(m, dst);
            const_cast<Impl*>(this)->h_present[m] = 1;
            const_cast<Impl*>(this)->t.d2h_bytes += view->group(M.group).image_bytes;
        }
        return dst;
    }

    uint32_t member_for(uint32_t batch) const {
        const int64_t m = view->member_of(batch);
        require(m >= 0, Errc::invalid_argument,
                "batch " + std::to_string(batch) + " is not a member of any group (routing bug)");
        return static_cast<uint32_t>(m);
    }

    const GpuContext::Kernel& resolve(uint32_t store_kernel, uint32_t node) const {
        const int32_t k = store_kernel < kernel_of.size() ? kernel_of[store_kernel] : -1;
        if (k < 0) {
            const KernelRef ref = view->kernel_ref(store_kernel);
            raise(Errc::unresolved_kernel, "node " + std::to_string(node) + " references " + ref.describe());
        }
        return *ctx->kernel_by_entry_id(static_cast<uint32_t>(k));
    }

    void restore_binaries();
    void open_binary(uint64_t hash, const KernelBinaryRecord& rec, uint32_t ordinal, KernelImage& image,
                     GpuContext::OpenedLibrary& opened);
    void build_group(uint32_t g);
    void prepare_kernels(uint32_t g, uint32_t m, bool load_functions = false);
    std::string shape_key(uint32_t g);
    uint64_t build_graph_for(uint32_t g, uint32_t m, CUgraph& graph, std::vector<CUgraphNode>& nodes);
    void kernel_params(const fdt_node& d, const uint8_t* blob, const GpuContext::Kernel& K,
                       CUDA_KERNEL_NODE_PARAMS& p, void** extra, size_t* size) const;
    CUDA_MEMCPY3D memcpy_params(const uint8_t* blob) const;
    CUDA_MEMSET_NODE_PARAMS memset_params(const uint8_t* blob) const;
    uint64_t safe(uint64_t addr) const;
    uint64_t apply_member(uint32_t g, uint32_t m);
    LaunchTrace replay(uint32_t batch);
};

// ---------------------------------------------------------------- restore

// restore_binaries (binary_catalog.cpp:200-227): every cataloged binary is
// checked, parsed and opened (cuLibraryLoadData + cuLibraryGetKernel) on
// `prepare_lanes` host threads — the driver's library load scales with
// threads — then registered and device-inited in catalog order on this one.
void ServingContext::Impl::restore_binaries() {
    struct Item {
        uint64_t hash;
        const KernelBinaryRecord* rec;
        uint32_t ordinal;
        KernelImage image;
        GpuContext::OpenedLibrary opened;
    };
    std::vector<Item> items;
    uint32_t ordinal = 0;
    for (const auto& [hash, rec] : catalog.binaries) {
        const uint32_t ord = ordinal++;
        if (ctx->has_library(hash)) continue;  // a second restore is a no-op
        items.push_back(Item{hash, &rec, ord, {}, {}});
    }
    unsigned lanes = std::max(1u, std::min(opts.prepare_lanes, 8u));
    if (const char* env = std::getenv("FOUNDRY_RESTORE_LANES")) lanes = std::max(1, std::atoi(env));
    std::vector<std::exception_ptr> failed(items.size());
    parallel_for(items.size(), lanes, [&](size_t i) {
        try {
            open_binary(items[i].hash, *items[i].rec, items[i].ordinal, items[i].image, items[i].opened);
        } catch (...) {
            failed[i] = std::current_exception();
        }
    });
    debug_phase("restore: libraries opened");
    // the first failure in catalog order is the one reported, as sequentially
    for (size_t i = 0; i < items.size(); ++i) {
        if (!failed[i]) continue;
        for (Item& it : items)
            if (it.opened.lib) driver().cuLibraryUnload(it.opened.lib);
        std::rethrow_exception(failed[i]);
    }
    for (Item& it : items) {
        const uint32_t lib = ctx->register_library(it.hash, it.image, std::move(it.opened), it.ordinal,
                                                   it.rec->needs_device_init);
        if (it.rec->needs_device_init && !opts.faults.skip_device_init) ctx->run_device_init(lib);
    }
}

void ServingContext::Impl::open_binary(uint64_t hash, const KernelBinaryRecord& rec, uint32_t ord,
                                       KernelImage& image_out, GpuContext::OpenedLibrary& opened) {
    {
        const std::string rel = "binaries/" + hex16(hash) + ".bin";
        std::vector<uint8_t> fetched;
        std::span<const uint8_t> payload;
        uint64_t digest = 0;
        if (staged->has(rel)) {
            payload = file_host(rel);
            digest = manifest.file_digests.at(rel);  // verified on the GPU by stage 2
        } else {
            fetched = slurp(ArchivePaths{root}.binary(hash));
            payload = fetched;
            digest = crc64(fetched);
        }
        require(digest == hash, Errc::archive_corruption,
                "binary " + hex16(hash) + " content does not match its hash");
        const KernelImage image = parse_kernel_image(payload);
        require(!image.relocatable, Errc::binary_format,
                "relocatable segment must be pre-linked before loading");
        const std::string crel = "binaries/" + hex16(hash) + ".sm_100a.cubin";
        std::vector<uint8_t> built;
        std::span<const uint8_t> cubin;
        if (staged->has(crel)) {
            cubin = file_host(crel);
        } else {  // reference-written archive: compile the trace module now
            built = compile_ptx_to_cubin(trace_module_ptx(image, ord, rec.needs_device_init));
            cubin = built;
        }
        opened = ctx->open_library(image, cubin);
        image_out = std::move(image);
    }
}

// ---------------------------------------------------------------- graph params

uint64_t ServingContext::Impl::safe(uint64_t addr) const {
    // memop nodes are constructed with live addresses only; an address outside
    // the mapping is reported at replay (unmapped-address) before any launch
    return ctx->physically_backed(addr) ? addr : ctx->backing_base();
}

void ServingContext::Impl::kernel_params(const fdt_node& d, const uint8_t* blob,
                                         const GpuContext::Kernel& K, CUDA_KERNEL_NODE_PARAMS& p,
                                         void** extra, size_t* size) const {
    std::memset(&p, 0, sizeof p);
    p.func = ctx->function(K);  // this context's function: it carries the launch limits set at LOAD
    p.gridDimX = d.grid[0];
    p.gridDimY = d.grid[1];
    p.gridDimZ = d.grid[2];
    p.blockDimX = d.block[0];
    p.blockDimY = d.block[1];
    p.blockDimZ = d.block[2];
    p.sharedMemBytes = d.shmem;
    *size = K.arg_buffer_size;  // the device ABI of the entry; extra bytes stay host-side
    extra[0] = CU_LAUNCH_PARAM_BUFFER_POINTER;
    extra[1] = const_cast<uint8_t*>(blob);
    extra[2] = CU_LAUNCH_PARAM_BUFFER_SIZE;
    extra[3] = size;
    extra[4] = CU_LAUNCH_PARAM_END;
    p.extra = extra;
}

CUDA_MEMCPY3D ServingContext::Impl::memcpy_params(const uint8_t* blob) const {
    CUDA_MEMCPY3D c;
    std::memset(&c, 0, sizeof c);
    c.srcMemoryType = CU_MEMORYTYPE_DEVICE;
    c.srcDevice = safe(rd64(blob));
    c.dstMemoryType = CU_MEMORYTYPE_DEVICE;
    c.dstDevice = safe(rd64(blob + 8));
    c.WidthInBytes = rd64(blob + 16);
    c.Height = 1;
    c.Depth = 1;
    require(c.WidthInBytes > 0, Errc::invalid_argument, "memcpy node with zero length");
    return c;
}

CUDA_MEMSET_NODE_PARAMS ServingContext::Impl::memset_params(const uint8_t* blob) const {
    CUDA_MEMSET_NODE_PARAMS m;
    std::memset(&m, 0, sizeof m);
    m.dst = safe(rd64(blob));
    const uint64_t value = rd64(blob + 8), len = rd64(blob + 16);
    require(len > 0, Errc::invalid_argument, "memset node with zero length");
    if (value <= 0xFF) {
        m.elementSize = 1;
        m.width = len;
    } else {
        require(value <= 0xFFFFFFFFull && len % 4 == 0, Errc::invalid_argument,
                "memset value " + std::to_string(value) + " is not representable by a device memset");
        m.elementSize = 4;
        m.width = len / 4;
    }
    m.value = static_cast<unsigned int>(value);
    m.height = 1;
    m.pitch = 0;
    return m;
}

// validate every kernel node before touching the driver (sim_driver.cpp:295-305)
// and apply the per-function launch limits its nodes need
void ServingContext::Impl::prepare_kernels(uint32_t gi, uint32_t m, bool load_functions) {
    const fdt_group& G = view->group(gi);
    const uint8_t* img = member_image(m);
    for (uint32_t n = 0; n < G.n_nodes; ++n) {
        fdt_node d;
        std::memcpy(&d, img + 48ull * n, sizeof d);
        if (d.type != 0) continue;
        const auto& K = resolve(d.kernel, n);
        require(d.blob_len >= K.arg_buffer_size, Errc::invalid_argument,
                "build_graph: argument buffer smaller than '" + K.name + "' declares (" +
                    std::to_string(d.blob_len) + " < " + std::to_string(K.arg_buffer_size) + ")");
        const FuncAttrs fa = view->kernel_func_attrs(d.kernel);
        const int want = std::max<int>(fa.max_dynamic_shared_size_bytes, static_cast<int>(d.shmem));
        if (want > 48 * 1024) ctx->require_dynamic_smem(K, want);
        if (fa.preferred_shared_memory_carveout >= 0) ctx->set_carveout(K, fa.preferred_shared_memory_carveout);
        if (load_functions) ctx->ensure_loaded(K);
    }
}

// What an instantiated exec fixes: node count and types, edges, and the launch
// attributes the template build applies. Groups with equal keys can share one
// exec (everything else is per-node parameters: cuGraphExec*NodeSetParams).
std::string ServingContext::Impl::shape_key(uint32_t gi) {
    const fdt_group& G = view->group(gi);
    const uint8_t* img = member_image(G.first_member);
    std::string key;
    auto put = [&](const void* p, size_t n) { key.append(static_cast<const char*>(p), n); };
    put(&G.n_nodes, 4);
    for (uint32_t n = 0; n < G.n_nodes; ++n) {
        fdt_node d;
        std::memcpy(&d, img + 48ull * n, sizeof d);
        put(&d.type, 1);
        if (d.type != 0) continue;
        const fdt_node_attrs& a = view->node_attrs(gi, n);
        const uint32_t csize = a.cluster[0] * a.cluster[1] * a.cluster[2];
        const bool cluster_ok = csize > 1 && csize <= 8 && d.grid[0] % a.cluster[0] == 0 &&
                                d.grid[1] % a.cluster[1] == 0 && d.grid[2] % a.cluster[2] == 0;
        const uint32_t applied[4] = {cluster_ok ? a.cluster[0] : 1u, cluster_ok ? a.cluster[1] : 1u,
                                     cluster_ok ? a.cluster[2] : 1u,
                                     (a.sched_policy > 0 && a.sched_policy <= 2) ? uint32_t(a.sched_policy) : 0u};
        put(applied, sizeof applied);
    }
    const auto e = view->edges(gi);
    put(e.data(), size_t(G.n_edges) * 2 * sizeof(uint32_t));
    return key;
}

uint64_t ServingContext::Impl::build_graph_for(uint32_t gi, uint32_t m, CUgraph& graph,
                                               std::vector<CUgraphNode>& nodes) {
    const DriverApi& api = driver();
    dev->make_current();
    const fdt_group& G = view->group(gi);
    const uint8_t* img = member_image(m);
    const uint8_t* pool = img + 48ull * G.n_nodes;
    uint64_t calls = 0;

    prepare_kernels(gi, m);

    cu_check(api.cuGraphCreate(&graph, 0), "cuGraphCreate");
    nodes.assign(G.n_nodes, nullptr);
    for (uint32_t n = 0; n < G.n_nodes; ++n) {
        fdt_node d;
        std::memcpy(&d, img + 48ull * n, sizeof d);
        const uint8_t* blob = pool + d.blob_off;
        CUgraphNode& node = nodes[n];
        switch (d.type) {
            case 0: {
                const auto& K = resolve(d.kernel, n);
                CUDA_KERNEL_NODE_PARAMS p;
                void* extra[5];
                size_t size;
                kernel_params(d, blob, K, p, extra, &size);
                cu_check(api.cuGraphAddKernelNode(&node, graph, nullptr, 0, &p), "cuGraphAddKernelNode");
                if (opts.device_updates) {
                    CUkernelNodeAttrValue v{};
                    v.deviceUpdatableKernelNode.deviceUpdatable = 1;
                    cu_check(api.cuGraphKernelNodeSetAttribute(node, CU_LAUNCH_ATTRIBUTE_DEVICE_UPDATABLE_KERNEL_NODE,
                                                               &v),
                             "cuGraphKernelNodeSetAttribute(device updatable)");
                }
                const fdt_node_attrs& a = view->node_attrs(gi, n);
                const bool non_default = a.cluster[0] != 1 || a.cluster[1] != 1 || a.cluster[2] != 1 ||
                                         a.sched_policy || a.sync_default || a.sync_remote || !a.attr_query;
                if (non_default) {
                    ++calls;
                    const uint32_t csize = a.cluster[0] * a.cluster[1] * a.cluster[2];
                    const bool cluster_ok = csize > 1 && csize <= 8 && d.grid[0] % a.cluster[0] == 0 &&
                                            d.grid[1] % a.cluster[1] == 0 && d.grid[2] % a.cluster[2] == 0;
                    if (cluster_ok) {
                        CUkernelNodeAttrValue v{};
                        v.clusterDim.x = a.cluster[0];
                        v.clusterDim.y = a.cluster[1];
                        v.clusterDim.z = a.cluster[2];
                        cu_check(api.cuGraphKernelNodeSetAttribute(node, CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION, &v),
                                 "cuGraphKernelNodeSetAttribute(cluster)");
                    }
                    if (a.sched_policy > 0 && a.sched_policy <= 2) {
                        CUkernelNodeAttrValue v{};
                        v.clusterSchedulingPolicyPreference =
                            static_cast<CUclusterSchedulingPolicy>(a.sched_policy);
                        cu_check(api.cuGraphKernelNodeSetAttribute(
                                     node, CU_LAUNCH_ATTRIBUTE_CLUSTER_SCHEDULING_POLICY_PREFERENCE, &v),
                                 "cuGraphKernelNodeSetAttribute(policy)");
                    }
                }
                break;
            }
            case 1: {
                const CUDA_MEMCPY3D c = memcpy_params(blob);
                cu_check(api.cuGraphAddMemcpyNode(&node, graph, nullptr, 0, &c, cu_ctx), "cuGraphAddMemcpyNode");
                break;
            }
            case 2: {
                const CUDA_MEMSET_NODE_PARAMS s = memset_params(blob);
                cu_check(api.cuGraphAddMemsetNode(&node, graph, nullptr, 0, &s, cu_ctx), "cuGraphAddMemsetNode");
                break;
            }
            default:
                cu_check(api.cuGraphAddEmptyNode(&node, graph, nullptr, 0), "cuGraphAddEmptyNode");
        }
        ++calls;
    }
    const auto e = view->edges(gi);
    if (G.n_edges) {
        std::vector<CUgraphNode> from(G.n_edges), to(G.n_edges);
        for (uint32_t i = 0; i < G.n_edges; ++i) {
            from[i] = nodes[e[2 * i]];
            to[i] = nodes[e[2 * i + 1]];
        }
        cu_check(api.cuGraphAddDependencies(graph, from.data(), to.data(), G.n_edges),
                 "cuGraphAddDependencies");
        calls += G.n_edges;
    }
    return calls;
}

void ServingContext::Impl::build_group(uint32_t gi) {
    const DriverApi& api = driver();
    const fdt_group& G = view->group(gi);
    Group& grp = groups[gi];
    const uint32_t m = G.first_member;  // representative: the smallest label
    const auto t0 = Clock::now();
    debug_phase("build group");
    build_graph_for(gi, m, grp.graph, grp.nodes);
    debug_phase("built group");
    const auto e = view->edges(gi);
    (void)e;
    // counters mirror the reference builder lane (sim_driver.cpp:307-313)
    ctx->c_add_node.fetch_add(G.n_nodes);
    ctx->c_add_edge.fetch_add(G.n_edges);
    for (uint32_t n = 0; n < G.n_nodes; ++n) {
        const fdt_node_attrs& a = view->node_attrs(gi, n);
        fdt_node d;
        std::memcpy(&d, member_image(m) + 48ull * n, sizeof d);
        if (d.type == 0 && (a.cluster[0] != 1 || a.cluster[1] != 1 || a.cluster[2] != 1 ||
                            a.sched_policy || a.sync_default || a.sync_remote || !a.attr_query))
            ctx->c_set_attr.fetch_add(1);
    }
    const double build = ms_since(t0);
    const auto t1 = Clock::now();
    cu_check(api.cuGraphInstantiate(&grp.exec, grp.graph, 0), "cuGraphInstantiate");
    debug_phase("instantiated group");
    ctx->c_instantiate.fetch_add(1);
    if (opts.device_updates) {  // device handles of the kernel nodes, what they were built with
        const uint8_t* img = member_image(m);
        grp.serve_nodes.assign(G.n_nodes, FdyServeNode{});
        grp.memops.assign(G.n_nodes, {0, 0, 0});
        for (uint32_t n = 0; n < G.n_nodes; ++n) {
            fdt_node d;
            std::memcpy(&d, img + 48ull * n, sizeof d);
            FdyServeNode& sn = grp.serve_nodes[n];
            if (d.type == 0) {
                CUkernelNodeAttrValue v{};
                cu_check(api.cuGraphKernelNodeGetAttribute(grp.nodes[n], CU_LAUNCH_ATTRIBUTE_DEVICE_UPDATABLE_KERNEL_NODE,
                                                           &v),
                         "cuGraphKernelNodeGetAttribute(device node)");
                sn.devnode = reinterpret_cast<void*>(v.deviceUpdatableKernelNode.devNode);
                sn.param_bytes = resolve(d.kernel, n).arg_buffer_size;
                sn.kernel = d.kernel;
                std::memcpy(sn.block, d.block, sizeof sn.block);
                sn.shmem = d.shmem;
            } else if (d.type == 1 || d.type == 2) {
                std::memcpy(grp.memops[n].data(), img + 48ull * G.n_nodes + d.blob_off, 24);
                sn.memop_slot = static_cast<int32_t>(grp.memop_nodes.size());
                grp.memop_nodes.push_back(n);
            }
            if (d.type != 1 && d.type != 2) sn.memop_slot = -1;
            if (d.type == 0) ++grp.n_kernel_nodes;
        }
        grp.d_serve_nodes = DeviceBuffer(*dev, sizeof(FdyServeNode) * std::max<uint32_t>(G.n_nodes, 1));
        cuda_check(cudaMemcpy(grp.d_serve_nodes.data(), grp.serve_nodes.data(), sizeof(FdyServeNode) * G.n_nodes,
                              cudaMemcpyHostToDevice),
                   "cudaMemcpy(serve table)");
        cu_check(api.cuGraphUpload(grp.exec, dev->stream()), "cuGraphUpload");
    }
    const double inst = ms_since(t1);
    if (std::getenv("FOUNDRY_DEBUG"))
        std::fprintf(stderr, "[foundry] group %u: %u nodes %u edges build %.3f ms instantiate %.3f ms\n", gi,
                     G.n_nodes, G.n_edges, build, inst);
    {
        std::lock_guard lock(stats_mu);  // builder lanes may run concurrently
        lane_acquisitions += 2;
        t.build_ms += build;
        t.instantiate_ms += inst;
    }
    grp.applied = m;
    grp.bound = gi;
}

// ---------------------------------------------------------------- serve

void ServingContext::Impl::build_serve_plan() {
    const uint32_t nm = view->n_members(), ng = static_cast<uint32_t>(groups.size());
    std::vector<uint64_t> off(nm);
    std::vector<uint32_t> grp_of(nm), base(nm);
    std::vector<const FdyServeNode*> tables(ng);
    std::vector<uint32_t> nn(ng);
    uint32_t slots = 0;
    for (uint32_t m = 0; m < nm; ++m) {
        const fdt_member& M = view->member(m);
        off[m] = M.out_off;
        grp_of[m] = M.group;
        base[m] = slots;
        slots += static_cast<uint32_t>(groups[M.group].memop_nodes.size());
    }
    for (uint32_t g = 0; g < ng; ++g) {
        tables[g] = reinterpret_cast<const FdyServeNode*>(groups[g].d_serve_nodes.data());
        nn[g] = view->group(g).n_nodes;
    }
    // one scratch buffer: offsets | groups | bases | tables | n_nodes | flags | records
    const size_t bytes = 8ull * nm + 4ull * nm + 4ull * nm + 8ull * ng + 4ull * ng + nm + 24ull * slots + 64;
    DeviceBuffer scratch(*dev, bytes);
    unsigned char* p = scratch.data();
    auto put = [&](const void* src, size_t n) {
        unsigned char* at = p;
        if (n) cuda_check(cudaMemcpyAsync(at, src, n, cudaMemcpyHostToDevice, dev->stream()), "serve plan H2D");
        p += (n + 7) / 8 * 8;
        return at;
    };
    FdyServePlanArgs a{};
    a.arena = d_members.data();
    a.member_off = reinterpret_cast<const uint64_t*>(put(off.data(), 8ull * nm));
    a.member_group = reinterpret_cast<const uint32_t*>(put(grp_of.data(), 4ull * nm));
    a.memop_base = reinterpret_cast<const uint32_t*>(put(base.data(), 4ull * nm));
    a.group_nodes = reinterpret_cast<const FdyServeNode* const*>(put(tables.data(), 8ull * ng));
    a.group_n_nodes = reinterpret_cast<const uint32_t*>(put(nn.data(), 4ull * ng));
    a.member_host = p;
    p += (nm + 7) / 8 * 8;
    a.records = reinterpret_cast<uint64_t*>(p);
    a.n_members = nm;
    cuda_check(fdy_launch_serve_plan(&a, dev->stream()), "serve plan launch");
    serve_member_host.assign(nm, 1);
    serve_error = PinnedBuffer(*dev, sizeof(uint32_t) + nm);
    std::memset(serve_error.data(), 0, sizeof(uint32_t) + nm);
    serve_plan_records.assign(slots, {0, 0, 0});
    if (nm) cuda_check(cudaMemcpyAsync(serve_member_host.data(), a.member_host, nm, cudaMemcpyDeviceToHost,
                                       dev->stream()), "serve plan D2H");
    if (slots) cuda_check(cudaMemcpyAsync(serve_plan_records.data(), a.records, 24ull * slots,
                                          cudaMemcpyDeviceToHost, dev->stream()), "serve plan D2H");
    cuda_check(cudaStreamSynchronize(dev->stream()), "cudaStreamSynchronize(serve plan)");
    serve_memop_base = std::move(base);
}

// device_updates serve: kernel nodes from the GPU (asynchronous: the launch is
// queued on the device stream ahead of the next graph launch), memop nodes from
// the host out of the LOAD-time plan. No readback. Returns the nodes updated, or
// kNoMember when the member needs the host path (function / block / shared
// memory of a node differs from what its template was built with).
uint64_t ServingContext::Impl::serve_on_device(uint32_t gi, uint32_t m) {
    if (serve_member_host[m]) return kNoMember;
    Group& grp = groups[gi];
    const fdt_group& G = view->group(gi);
    const DriverApi& api = driver();
    dev->make_current();
    FdyServeArgs a{};
    a.nodes = reinterpret_cast<const FdyServeNode*>(grp.d_serve_nodes.data());
    a.image = d_members.data() + view->member(m).out_off;
    a.n_nodes = G.n_nodes;  // host_flags / host_records null: nothing comes back
    a.member = m;
    a.error_word = reinterpret_cast<uint32_t*>(serve_error.data());
    a.member_failed = serve_error.data() + sizeof(uint32_t);
    a.inject_failure = opts.faults.fail_device_serve ? 1u : 0u;
    cuda_check(fdy_launch_serve(&a, dev->stream()), "serve kernel launch");
    uint64_t touched = grp.n_kernel_nodes;
    for (uint32_t k = 0; k < grp.memop_nodes.size(); ++k) {
        const uint32_t n = grp.memop_nodes[k];
        const std::array<uint64_t, 3>& rec = serve_plan_records[serve_memop_base[m] + k];
        if (rec == grp.memops[n]) continue;
        const uint8_t* blob = reinterpret_cast<const uint8_t*>(rec.data());
        CUgraphNodeType t;
        cu_check(api.cuGraphNodeGetType(grp.nodes[n], &t), "cuGraphNodeGetType");
        if (t == CU_GRAPH_NODE_TYPE_MEMCPY) {
            const CUDA_MEMCPY3D c = memcpy_params(blob);
            cu_check(api.cuGraphExecMemcpyNodeSetParams(grp.exec, grp.nodes[n], &c, cu_ctx),
                     "cuGraphExecMemcpyNodeSetParams");
        } else {
            const CUDA_MEMSET_NODE_PARAMS sp = memset_params(blob);
            cu_check(api.cuGraphExecMemsetNodeSetParams(grp.exec, grp.nodes[n], &sp, cu_ctx),
                     "cuGraphExecMemsetNodeSetParams");
        }
        grp.memops[n] = rec;
        ++touched;
    }
    return touched;
}

// Called with the device stream synchronized. A failed device update marks its
// member for the host path (every later serve of it goes through the host) and,
// if its exec still holds that member, forgets it, so the next apply
// re-applies every node on the host. True when the exec of group gi was
// affected.
bool ServingContext::Impl::recover_device_serve(uint32_t gi) {
    if (serve_error.size() == 0) return false;
    volatile uint32_t* any = reinterpret_cast<volatile uint32_t*>(serve_error.data());
    if (*any == 0) return false;
    *any = 0;
    volatile uint8_t* failed = serve_error.data() + sizeof(uint32_t);
    bool mine = false;
    for (uint32_t m = 0; m < serve_member_host.size(); ++m) {
        if (!failed[m]) continue;
        failed[m] = 0;
        serve_member_host[m] = 1;
        for (Group& g : groups) {
            if (g.applied != m) continue;
            g.applied = kNoMember;
            mine = mine || &g == &exec_of(gi);
        }
    }
    return mine;
}

uint64_t ServingContext::Impl::apply_member(uint32_t gi, uint32_t m) {
    Group& grp = exec_of(gi);
    if (grp.applied == m) return 0;
    if (opts.device_updates && !grp.serve_nodes.empty()) {
        const uint64_t touched = serve_on_device(gi, m);
        if (touched == kNoMember) grp.applied = kNoMember;  // the host path applies every node
        if (touched != kNoMember) {
            grp.applied = m;
            grp.bound = gi;
            ++lane_acquisitions;
            ctx->c_update.fetch_add(1);
            ctx->c_update_touched.fetch_add(touched);
            return touched;
        }
    }
    const DriverApi& api = driver();
    dev->make_current();
    const fdt_group& G = view->group(gi);
    const uint8_t* img = member_image(m);
    const uint8_t* pool = img + 48ull * G.n_nodes;
    // what the exec holds now: a member of this group, or (share_execs) of
    // another group of the same shape, whose image layout may differ
    const uint8_t* cur = grp.applied == kNoMember ? nullptr : member_image(grp.applied);
    const uint8_t* cur_pool = cur ? cur + 48ull * view->group(grp.bound).n_nodes : nullptr;
    uint64_t touched = 0;
    for (uint32_t n = 0; n < G.n_nodes; ++n) {
        fdt_node d;
        std::memcpy(&d, img + 48ull * n, sizeof d);
        const uint8_t* blob = pool + d.blob_off;
        if (cur) {
            fdt_node c;
            std::memcpy(&c, cur + 48ull * n, sizeof c);
            // descriptor up to blob_off (type, kernel, dims, shmem, blob_len), then the bytes
            const bool same = std::memcmp(&c, &d, offsetof(fdt_node, blob_off)) == 0 &&
                              std::memcmp(cur_pool + c.blob_off, blob, d.blob_len) == 0;
            if (same) continue;
        }
        ++touched;
        switch (d.type) {
            case 0: {
                const auto& K = resolve(d.kernel, n);
                require(d.blob_len >= K.arg_buffer_size, Errc::invalid_argument,
                        "exec_update: argument buffer smaller than '" + K.name + "' declares");
                CUDA_KERNEL_NODE_PARAMS p;
                void* extra[5];
                size_t size;
                kernel_params(d, blob, K, p, extra, &size);
                cu_check(api.cuGraphExecKernelNodeSetParams(grp.exec, grp.nodes[n], &p),
                         "cuGraphExecKernelNodeSetParams");
                break;
            }
            case 1: {
                const CUDA_MEMCPY3D c = memcpy_params(blob);
                cu_check(api.cuGraphExecMemcpyNodeSetParams(grp.exec, grp.nodes[n], &c, cu_ctx),
                         "cuGraphExecMemcpyNodeSetParams");
                break;
            }
            case 2: {
                const CUDA_MEMSET_NODE_PARAMS s = memset_params(blob);
                cu_check(api.cuGraphExecMemsetNodeSetParams(grp.exec, grp.nodes[n], &s, cu_ctx),
                         "cuGraphExecMemsetNodeSetParams");
                break;
            }
            default: break;
        }
    }
    if (opts.device_updates && !grp.serve_nodes.empty()) {
        // host updates of device-updatable nodes take effect after an upload
        cu_check(api.cuGraphUpload(grp.exec, dev->stream()), "cuGraphUpload");
        for (uint32_t n = 0; n < G.n_nodes; ++n) {
            fdt_node d;
            std::memcpy(&d, img + 48ull * n, sizeof d);
            if (d.type == 1 || d.type == 2) std::memcpy(grp.memops[n].data(), pool + d.blob_off, 24);
        }
    }
    grp.applied = m;
    grp.bound = gi;
    ++lane_acquisitions;
    ctx->c_update.fetch_add(1);
    ctx->c_update_touched.fetch_add(touched);
    return touched;
}

// ---------------------------------------------------------------- replay

LaunchTrace ServingContext::Impl::replay(uint32_t batch) {
    const uint32_t m = member_for(batch);
    const uint32_t gi = view->member(m).group;
    apply_member(gi, m);
    const fdt_group& G = view->group(gi);
    const uint8_t* img = member_image(m);
    const uint8_t* pool = img + 48ull * G.n_nodes;

    // host pre-validation in node order (reference replay, sim_driver.cpp:423-470)
    LaunchTrace trace;
    trace.records.reserve(G.n_nodes);
    struct Expect {
        uint32_t node;
        const GpuContext::Kernel* k;
        const fdt_node* d;
        const uint8_t* blob;
    };
    std::vector<fdt_node> descs(G.n_nodes);
    std::vector<Expect> expect;
    auto check_mapped = [&](uint32_t node, uint32_t off, uint64_t a) {
        require(ctx->address_mapped(a), Errc::unmapped_address,
                "node " + std::to_string(node) + " offset " + std::to_string(off) +
                    " references unmapped address 0x" + hex16(a));
    };
    for (uint32_t n = 0; n < G.n_nodes; ++n) {
        fdt_node& d = descs[n];
        std::memcpy(&d, img + 48ull * n, sizeof d);
        const uint8_t* blob = pool + d.blob_off;
        TraceRecord r;
        r.node_id = n;
        r.type = static_cast<NodeType>(d.type);
        if (d.type == 0) {
            const auto& K = resolve(d.kernel, n);
            require(!ctx->library_requires_init(K.library) || ctx->library_device_inited(K.library),
                    Errc::device_state_uninitialized,
                    "node " + std::to_string(n) + " kernel '" + K.name + "' used before device-side init");
            require(d.blob_len >= K.arg_buffer_size, Errc::invalid_argument,
                    "replay: argument buffer smaller than '" + K.name + "' declares (" +
                        std::to_string(d.blob_len) + " < " + std::to_string(K.arg_buffer_size) + ")");
            for (uint32_t off : K.hidden_offsets) {
                const uint64_t a = rd64(blob + off);
                check_mapped(n, off, a);
                r.addresses.push_back(a);
            }
            r.kernel_name = K.name;
            r.grid = {d.grid[0], d.grid[1], d.grid[2]};
            r.block = {d.block[0], d.block[1], d.block[2]};
            r.shared_mem_bytes = d.shmem;
            r.arg_digest = crc64(blob, d.blob_len);
            expect.push_back({n, &K, &descs[n], blob});
        } else if (d.type == 1 || d.type == 2) {
            const uint64_t a0 = rd64(blob), a1 = rd64(blob + 8);
            check_mapped(n, 0, a0);
            if (d.type == 1) {
                check_mapped(n, 8, a1);
                r.addresses = {a0, a1};
            } else {
                r.addresses = {a0};
            }
            r.arg_digest = crc64(blob, 24);
        }
        trace.records.push_back(std::move(r));
    }

    // launch the instantiated graph and verify the device-side trace
    const DriverApi& api = driver();
    dev->make_current();
    ctx->reset_trace();
    cu_check(api.cuGraphLaunch(exec_of(gi).exec, dev->stream()), "cuGraphLaunch");
    ctx->c_replay.fetch_add(1);
    dev->sync();
    // a device serve that failed left its exec with stale parameters: re-apply
    // that member on the host and, if it is this batch's, launch again
    if (recover_device_serve(gi)) return replay(batch);
    if (!opts.verify_replay) return trace;
    const std::vector<uint8_t> recs = ctx->read_trace();
    // index the expected launches by (entry id, parameter bytes)
    std::multimap<std::pair<uint32_t, uint64_t>, const Expect*> want;
    for (const auto& e : expect)
        want.emplace(std::make_pair(e.k->entry_id, crc64(e.blob, e.k->arg_buffer_size)), &e);
    size_t at = 0, seen = 0;
    while (at + FDY_TRACE_HEADER_BYTES <= recs.size()) {
        fdy_trace_header h;
        std::memcpy(&h, recs.data() + at, sizeof h);
        require(h.magic == FDY_TRACE_MAGIC, Errc::cuda_error, "replay verification: torn trace record");
        const uint8_t* bytes = recs.data() + at + FDY_TRACE_HEADER_BYTES;
        auto range = want.equal_range({h.entry_id, crc64(bytes, h.n_bytes)});
        const Expect* hit = nullptr;
        for (auto it = range.first; it != range.second; ++it) {
            const Expect* e = it->second;
            if (e->k->arg_buffer_size == h.n_bytes && std::memcmp(e->blob, bytes, h.n_bytes) == 0 &&
                e->d->grid[0] == h.grid[0] && e->d->grid[1] == h.grid[1] && e->d->grid[2] == h.grid[2] &&
                e->d->block[0] == h.block[0] && e->d->block[1] == h.block[1] &&
                e->d->block[2] == h.block[2] && e->d->shmem == h.dyn_smem) {
                hit = e;
                want.erase(it);
                break;
            }
        }
        require(hit != nullptr, Errc::cuda_error,
                "replay verification: device launch of entry " + std::to_string(h.entry_id) +
                    " matches no expected node of batch " + std::to_string(batch));
        require(!(h.flags & FDY_TRACE_FLAG_UNINIT), Errc::device_state_uninitialized,
                "node " + std::to_string(hit->node) + " kernel '" + hit->k->name +
                    "' used before device-side init");
        require(!(h.flags & FDY_TRACE_FLAG_UNMAPPED), Errc::unmapped_address,
                "node " + std::to_string(hit->node) + " dereferenced an unmapped address on the device");
        at += FDY_TRACE_HEADER_BYTES + ((h.n_bytes + 15u) & ~15u);
        ++seen;
    }
    require(seen == expect.size() && want.empty(), Errc::cuda_error,
            "replay verification: " + std::to_string(seen) + " device launches recorded, " +
                std::to_string(expect.size()) + " kernel nodes expected");
    return trace;
}

// ---------------------------------------------------------------- load

namespace {

void verify_init_records(const std::vector<AllocationRecord>& actual, uint64_t actual_base,
                         const MemoryEventLog& log) {
    std::vector<AllocationRecord> expected;
    for (const auto& r : log.records)
        if (r.window == AllocWindow::pre_capture) expected.push_back(r);
    require(actual.size() == expected.size(), Errc::layout_divergence,
            "LOAD issued " + std::to_string(actual.size()) + " pre-window allocations, SAVE recorded " +
                std::to_string(expected.size()));
    for (size_t i = 0; i < expected.size(); ++i) {
        const bool same = actual[i].sequence == expected[i].sequence &&
                          actual[i].size == expected[i].size && actual[i].length == expected[i].length &&
                          actual[i].address - actual_base == expected[i].address - log.config.base;
        require(same, Errc::layout_divergence,
                "allocation sequence diverged at record " + std::to_string(i) + " (requested " +
                    std::to_string(actual[i].size) + " bytes at 0x" + hex16(actual[i].address) +
                    ", SAVE recorded " + std::to_string(expected[i].size) + " at 0x" +
                    hex16(expected[i].address) + ")");
    }
}

}  // namespace

ServingContext load(Device& device, const fs::path& archive, const LoadOptions& opts) {
    const auto t_all = Clock::now();
    require(opts.world >= 1 && opts.rank < opts.world, Errc::invalid_argument,
            "rank " + std::to_string(opts.rank) + " is outside world size " + std::to_string(opts.world));
    auto impl = std::make_unique<ServingContext::Impl>();
    // one LOAD at a time per process (see driver_lane()); declared after the
    // context, so on an exception the lane is released before ~Impl takes it
    std::unique_lock lane(driver_lane());
    auto& I = *impl;
    I.dev = &device;
    I.opts = opts;
    require(!(opts.share_execs && opts.device_updates), Errc::invalid_argument,
            "share_execs and device_updates exclude each other (a shared exec changes functions; "
            "device-updatable graphs cannot)");
    I.root = archive;
    ArchivePaths paths{archive};
    require(fs::exists(paths.manifest()), Errc::archive_corruption, "no manifest under " + archive.string());

    auto t0 = Clock::now();
    {
        const auto mb = slurp(paths.manifest());
        I.manifest = parse_manifest(std::string(mb.begin(), mb.end()));
    }
    I.t.manifest_ms = ms_since(t0);
    device.make_current();
    cu_check(driver().cuCtxGetCurrent(&I.cu_ctx), "cuCtxGetCurrent");
    I.ctx = std::make_unique<GpuContext>(device);
    debug_phase("gpu context ready");

    // 1. stage every listed file into HBM (reads overlap the DMA),
    // 2. stage + verify every digest: the store goes to HBM (GPU CRC as it
    //    lands); files LOAD parses stay in host memory; graphs.bin is only
    //    hashed when the store replaces it
    StageTimings st;
    std::future<PatchView> patch_view;  // reference-written archive: parsed while the rest streams
    try {
        StagePlan plan;
        const bool has_store = I.manifest.file_digests.count("templates.fdt") != 0;
        // the store goes to HBM; a reference-written archive's graphs.bin goes
        // there instead, for the GPU packer, with patch.bin read first
        plan.device = {has_store ? "templates.fdt" : "graphs.bin"};
        if (!has_store) plan.host_first = {"patch.bin"};
        plan.keep_host = [has_store](const std::string& rel) { return !(has_store && rel == "graphs.bin"); };
        I.staged = std::make_unique<StagedArchive>(device, archive, I.manifest, opts.prepare_lanes, &st, plan);
        if (!has_store && I.staged->has("patch.bin")) {
            StagedArchive* staged = I.staged.get();  // its errors surface in the packer, after integrity
            patch_view = std::async(std::launch::async, [staged] { return parse_patch_view(staged->host("patch.bin")); });
        }
        I.staged->verify(I.manifest, &st);
    } catch (const Error&) {
        rethrow_in_step("archive integrity");
    }
    I.t.stage_ms = st.read_ms;
    I.t.integrity_ms = st.integrity_ms;
    I.t.crc_kernel_ms = st.crc_kernel_ms;
    I.t.h2d_bytes += st.h2d_bytes;
    debug_phase("integrity done");

    const WorkloadSpec spec = WorkloadSpec::parse_text(I.manifest.workload_text);
    require(spec.digest() == I.manifest.workload_digest, Errc::archive_corruption,
            "embedded workload text does not match its recorded digest");
    I.catalog = parse_catalog(I.file_host("catalog.bin"));
    (void)parse_patch_view(I.file_host("patch.bin"));  // format check; the store carries the ops
    const MemoryEventLog log = parse_event_log(I.file_host("memlayout.bin"));

    // template store: packed offline (templates.fdt) or, for a reference-written
    // archive, packed now on the GPU from graphs.bin (in HBM) + patch.bin
    if (I.staged->has("templates.fdt")) {
        I.store_host = I.file_host("templates.fdt");
        I.view = std::make_unique<StoreView>(I.store_host);
        I.dstore = adopt_store(device, I.staged->device("templates.fdt"), I.store_host.size(),
                               I.view->header());
    } else {
        const auto t_pack = Clock::now();
        DevicePackResult packed;
        try {
            I.staged->order_after("graphs.bin", device.stream());
            packed = pack_template_store_device(
                device, I.file_host("graphs.bin"), I.staged->device("graphs.bin"), I.file_host("patch.bin"),
                I.manifest,
                I.staged->has("comm_slots.bin") ? I.file_host("comm_slots.bin") : std::span<const uint8_t>{},
                nullptr, nullptr, /*full_host_copy=*/false, &I.manifest.file_digests.at("graphs.bin"),
                patch_view.valid() ? &patch_view : nullptr);
        } catch (const Error&) {
            rethrow_in_step("template construction");
        }
        I.inline_store = std::move(packed.host_bytes);
        I.store_host = {I.inline_store.get(), packed.host_size};
        I.view = std::make_unique<StoreView>(I.store_host);
        I.dstore = adopt_store(device, packed.blob.data(), packed.host_size, I.view->header());
        I.dstore.blob = std::move(packed.blob);
        I.t.pack_ms = ms_since(t_pack);
    }
    const fdt_header& H = I.view->header();
    check_store_sources(H, I.manifest);
    require(opts.comm_values.size() >= H.n_values, Errc::invalid_argument,
            "the archive's comm slots read " + std::to_string(H.n_values) + " per-rank values, " +
                std::to_string(opts.comm_values.size()) + " given (LoadOptions::comm_values)");

    // 3. restore binaries (cuLibraryLoadData)
    t0 = Clock::now();
    if (!opts.faults.skip_binary_restore) {
        try {
            I.restore_binaries();
        } catch (const Error&) {
            rethrow_in_step("binary restore");
        }
    }
    I.kernel_of.assign(H.n_kernels, -1);
    for (uint32_t k = 0; k < H.n_kernels; ++k) {
        const auto* K = I.ctx->find_kernel(I.view->kernel(k).binary_hash, I.view->kernel_name(k));
        if (K) I.kernel_of[k] = static_cast<int32_t>(K->entry_id);
    }
    I.t.restore_ms = ms_since(t0);
    debug_phase("restore done");

    // 4. region
    t0 = Clock::now();
    RegionConfig cfg = I.manifest.allocator;
    cfg.base += static_cast<uint64_t>(opts.faults.base_shift_granules) * cfg.granularity;
    I.ctx->reserve_region(cfg, I.manifest.final_offset + cfg.granularity, opts.relocate);
    if (opts.preallocate) I.ctx->preallocate(I.manifest.final_offset);
    if (opts.faults.extra_prewindow_alloc) I.ctx->allocate(1);
    I.t.region_ms = ms_since(t0);
    debug_phase("region done");

    // 5. materialize every member for this rank: one fused kernel, then D2H
    t0 = Clock::now();
    MaterializeRequest req;
    req.rank = opts.rank;
    req.world = opts.world;
    req.values = opts.comm_values;
    const uint64_t new_base = I.ctx->region_base();
    req.new_base = (opts.relocate && new_base != I.manifest.allocator.base) ? new_base : 0;
    I.t.relocation_delta = req.new_base ? req.new_base - I.manifest.allocator.base : 0;
    I.d_members = DeviceBuffer(device, std::max<uint64_t>(H.members_image_bytes, 16));
    I.h_members.reset(new uint8_t[std::max<uint64_t>(H.members_image_bytes, 16)]);
    I.h_present.assign(H.n_members, 0);
    MaterializeTiming mt;
    mt.gate = false;  // inside LOAD: no stream hold for the events
    launch_materialize(device, I.dstore, req, I.d_members.data(), &mt);
    I.t.materialize_kernel_ms = mt.kernel_ms;
    I.t.materialize_ms = ms_since(t0);
    debug_phase("materialize done");
    t0 = Clock::now();
    for (uint32_t g = 0; g < H.n_groups; ++g) I.member_image(I.view->group(g).first_member);  // templates
    I.t.download_ms = ms_since(t0);
    debug_phase("download done");
    I.t.member_bytes = H.members_image_bytes;
    I.t.store_bytes = I.dstore.bytes;

    // 6. template construction (builder thread) || foreground init + window replay
    I.groups.resize(H.n_groups);
    std::exception_ptr builder_error, foreground_error;
    // builder lanes: templates are independent graphs; FOUNDRY_BUILD_LANES
    // host threads construct + instantiate them (1 = the reference's single lane)
    unsigned build_lanes = 1;
    if (const char* env = std::getenv("FOUNDRY_BUILD_LANES")) build_lanes = std::max(1, std::atoi(env));
    // (the driver loads each kernel's function lazily when its first node is
    // added; a separate loader thread ahead of the builder measured no gain:
    // function loads and instantiation serialize inside the driver)
    debug_phase("templates downloaded");
    if (opts.share_execs) {  // one exec per graph shape; the first group of a shape owns it
        std::map<std::string, uint32_t> first_of_shape;
        I.owner.resize(H.n_groups);
        for (uint32_t g = 0; g < H.n_groups; ++g)
            I.owner[g] = first_of_shape.emplace(I.shape_key(g), g).first->second;
        debug_phase("shape keys");
    }
    std::thread builder([&] {
        try {
            parallel_for(H.n_groups, build_lanes, [&](size_t g) {
                const uint32_t gi = static_cast<uint32_t>(g);
                if (I.owner.empty() || I.owner[gi] == gi) {
                    I.build_group(gi);
                    return;
                }
                // served through the owner's exec: its functions are loaded now, as
                // a build would (every template is servable when LOAD returns)
                const auto tf = Clock::now();
                debug_phase("function loads of a shared-exec template");
                I.prepare_kernels(gi, I.view->group(gi).first_member, /*load_functions=*/true);
                std::lock_guard lock(I.stats_mu);
                I.t.function_load_ms += ms_since(tf);
            });
        } catch (...) {
            builder_error = std::current_exception();
        }
    });
    t0 = Clock::now();
    try {
        try {
            std::vector<uint64_t> slot;
            for (const InitStep& st : build_init_plan(spec)) {
                if (st.kind == InitStep::Kind::alloc) {
                    if (st.slot >= slot.size()) slot.resize(st.slot + 1, 0);
                    slot[st.slot] = I.ctx->allocate(st.size);
                } else {
                    require(st.slot < slot.size(), Errc::invalid_argument, "init plan releases an unknown slot");
                    I.ctx->free(slot[st.slot]);
                }
            }
            verify_init_records(I.ctx->records(), I.ctx->region_base(), log);
        } catch (const Error&) {
            rethrow_in_step("foreground init");
        }
        try {
            I.ctx->replay_capture_window(log);
        } catch (const Error&) {
            rethrow_in_step("capture-window replay");
        }
    } catch (...) {
        foreground_error = std::current_exception();
    }
    I.t.foreground_ms = ms_since(t0);
    debug_phase("foreground done");
    builder.join();
    debug_phase("templates servable");
    if (foreground_error) std::rethrow_exception(foreground_error);
    if (builder_error) {
        try {
            std::rethrow_exception(builder_error);
        } catch (const Error&) {
            rethrow_in_step("template construction");
        }
    }

    if (opts.device_updates) I.build_serve_plan();

    // trace arena: one record (64 B + parameter bytes) per kernel node
    uint64_t arena = 1 << 16;
    for (uint32_t g = 0; g < H.n_groups; ++g)
        arena = std::max<uint64_t>(arena, I.view->group(g).image_bytes + 64ull * I.view->group(g).n_nodes);
    I.ctx->ensure_trace_arena(arena);
    I.ctx->sync_trace_state();
    lane.unlock();

    for (uint32_t m = 0; m < H.n_members; ++m) I.labels.push_back(I.view->member(m).label);
    std::sort(I.labels.begin(), I.labels.end());
    I.t.graphs = H.n_members;
    I.t.nodes = H.total_nodes;
    I.t.templates = H.n_groups;
    I.t.total_ms = ms_since(t_all);
    debug_phase("load returns");
    if (std::getenv("FOUNDRY_DEBUG")) std::fprintf(stderr, "[foundry] driver calls: %s\n", driver_call_stats(true).c_str());
    return ServingContext(std::move(impl));
}

namespace {
// Asks the kernel to read every manifest-listed file ahead (posix_fadvise
// WILLNEED: asynchronous readahead), so a LOAD whose archive is not in the page
// cache reads it while the CUDA context is being created. Best effort.
void prefetch_archive(const fs::path& archive) {
    try {
        const auto mb = slurp(ArchivePaths{archive}.manifest());
        const Manifest m = parse_manifest(std::string(mb.begin(), mb.end()));
        for (const auto& [rel, digest] : m.file_digests) {
            (void)digest;
            const int fd = ::open((archive / rel).c_str(), O_RDONLY | O_CLOEXEC);
            if (fd < 0) continue;
            ::posix_fadvise(fd, 0, 0, POSIX_FADV_WILLNEED);
            ::close(fd);
        }
    } catch (...) {
    }
}
}  // namespace

ServingContext load(const fs::path& archive, const LoadOptions& opts) {
    prefetch_archive(archive);
    debug_phase("archive readahead requested");
    debug_phase("open device");
    auto dev = std::make_unique<Device>(opts.device);
    debug_phase("device open");
    ServingContext sc = load(*dev, archive, opts);
    sc.impl_->owned_dev = std::move(dev);
    return sc;
}

// ---------------------------------------------------------------- ServingContext

ServingContext::ServingContext(std::unique_ptr<Impl> impl) : impl_(std::move(impl)) {}
ServingContext::ServingContext(ServingContext&&) noexcept = default;
ServingContext& ServingContext::operator=(ServingContext&&) noexcept = default;
ServingContext::~ServingContext() {
    if (impl_) {
        auto owned = std::move(impl_->owned_dev);
        impl_.reset();  // graphs/libraries/VA go before the device they live on
    }
}

LaunchTrace ServingContext::replay(uint32_t batch) { return impl_->replay(batch); }
std::vector<uint32_t> ServingContext::batches() const { return impl_->labels; }
const Manifest& ServingContext::manifest() const { return impl_->manifest; }
std::vector<AllocationRecord> ServingContext::allocation_records() const { return impl_->ctx->records(); }
GpuContext& ServingContext::context() { return *impl_->ctx; }
const LoadTimings& ServingContext::timings() const { return impl_->t; }
uint32_t ServingContext::template_count() const { return impl_->manifest.grouping.template_count; }

CounterSnapshot ServingContext::counters() const {
    CounterSnapshot s = impl_->ctx->counters();
    s["driver.lane_acquisitions"] = impl_->lane_acquisitions;
    s["driver.lane_contention_units"] = 0;
    s["catalog.prelink_calls"] = 0;
    s["catalog.linked_segments"] = 0;
    return s;
}

CapturedGraph ServingContext::prepared_params(uint32_t batch) const {
    const uint32_t m = impl_->member_for(batch);
    const auto& G = impl_->view->group(impl_->view->member(m).group);
    return impl_->view->image_to_graph(m, {impl_->member_image(m), G.image_bytes});
}

uint64_t ServingContext::serve(uint32_t batch) {
    const uint32_t m = impl_->member_for(batch);
    return impl_->apply_member(impl_->view->member(m).group, m);
}

namespace {
// canonical form of a trace arena: records sorted by (entry id, bytes)
std::vector<std::string> canonical_records(const std::vector<uint8_t>& recs) {
    std::vector<std::string> out;
    size_t at = 0;
    while (at + FDY_TRACE_HEADER_BYTES <= recs.size()) {
        fdy_trace_header h;
        std::memcpy(&h, recs.data() + at, sizeof h);
        const size_t len = FDY_TRACE_HEADER_BYTES + ((h.n_bytes + 15u) & ~15u);
        // meaningful fields only: header words before the pad, then the parameter bytes
        std::string r(reinterpret_cast<const char*>(recs.data() + at), offsetof(fdy_trace_header, magic));
        r.append(reinterpret_cast<const char*>(recs.data() + at + FDY_TRACE_HEADER_BYTES),
                 std::min<size_t>(h.n_bytes, recs.size() - at - FDY_TRACE_HEADER_BYTES));
        out.push_back(std::move(r));
        at += len;
    }
    std::sort(out.begin(), out.end());
    return out;
}
}  // namespace

bool ServingContext::fresh_capture_check(uint32_t batch, std::string* report) {
    Impl& I = *impl_;
    const DriverApi& api = driver();
    const uint32_t m = I.member_for(batch);
    const uint32_t gi = I.view->member(m).group;
    GpuContext& ctx = *I.ctx;
    Device& dev = *I.dev;
    cudaStream_t st = dev.stream();
    auto region_crc = [&]() {
        const Segment seg{0, ctx.backed_bytes()};
        return crc64_device(dev, reinterpret_cast<const unsigned char*>(ctx.backing_base()),
                            std::span<const Segment>(&seg, 1))[0];
    };
    // (a) the materialized exec
    I.replay(batch);  // validates addresses, applies member b
    ctx.zero_region();
    ctx.reset_trace();
    cu_check(api.cuGraphLaunch(I.exec_of(gi).exec, st), "cuGraphLaunch");
    dev.sync();
    const auto trace_a = canonical_records(ctx.read_trace());
    const uint64_t crc_a = region_crc();

    // (b) a fresh stream capture of the same launches, in capture (node) order
    const fdt_group& G = I.view->group(gi);
    const uint8_t* img = I.member_image(m);
    const uint8_t* pool = img + 48ull * G.n_nodes;
    ctx.zero_region();
    ctx.reset_trace();
    dev.sync();
    cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    for (uint32_t n = 0; n < G.n_nodes; ++n) {
        fdt_node d;
        std::memcpy(&d, img + 48ull * n, sizeof d);
        const uint8_t* blob = pool + d.blob_off;
        if (d.type == 0) {
            const auto& K = I.resolve(d.kernel, n);
            size_t size = K.arg_buffer_size;
            void* extra[5] = {CU_LAUNCH_PARAM_BUFFER_POINTER, const_cast<uint8_t*>(blob),
                              CU_LAUNCH_PARAM_BUFFER_SIZE, &size, CU_LAUNCH_PARAM_END};
            cu_check(api.cuLaunchKernel(ctx.function(K), d.grid[0], d.grid[1], d.grid[2], d.block[0], d.block[1],
                                        d.block[2], d.shmem, st, nullptr, extra),
                     "cuLaunchKernel(capture)");
        } else if (d.type == 1) {
            cuda_check(cudaMemcpyAsync(reinterpret_cast<void*>(rd64(blob + 8)),
                                       reinterpret_cast<const void*>(rd64(blob)), rd64(blob + 16),
                                       cudaMemcpyDeviceToDevice, st),
                       "cudaMemcpyAsync(capture)");
        } else if (d.type == 2) {
            const uint64_t value = rd64(blob + 8), len = rd64(blob + 16);
            if (value <= 0xFF)
                cu_check(api.cuMemsetD8Async(rd64(blob), static_cast<unsigned char>(value), len, st),
                         "cuMemsetD8Async(capture)");
            else
                cu_check(api.cuMemsetD32Async(rd64(blob), static_cast<unsigned int>(value), len / 4, st),
                         "cuMemsetD32Async(capture)");
        }
    }
    cudaGraph_t g = nullptr;
    cuda_check(cudaStreamEndCapture(st, &g), "cudaStreamEndCapture");
    cudaGraphExec_t x = nullptr;
    cuda_check(cudaGraphInstantiate(&x, g, 0), "cudaGraphInstantiate(capture)");
    cuda_check(cudaGraphLaunch(x, st), "cudaGraphLaunch(capture)");
    dev.sync();
    const auto trace_b = canonical_records(ctx.read_trace());
    const uint64_t crc_b = region_crc();
    cudaGraphExecDestroy(x);
    cudaGraphDestroy(g);
    const bool ok = trace_a == trace_b && crc_a == crc_b && !trace_a.empty();
    if (report)
        *report = "records " + std::to_string(trace_a.size()) + "/" + std::to_string(trace_b.size()) +
                  " region crc " + hex16(crc_a) + "/" + hex16(crc_b) + (ok ? " match" : " MISMATCH");
    return ok;
}

CapturedGraph ServingContext::capture_graph(uint32_t batch) {
    Impl& I = *impl_;
    const DriverApi& api = driver();
    const uint32_t m = I.member_for(batch);
    const uint32_t gi = I.view->member(m).group;
    const fdt_group& G = I.view->group(gi);
    const uint8_t* img = I.member_image(m);
    const uint8_t* pool = img + 48ull * G.n_nodes;
    // predecessors of every node, from the template's edges
    std::vector<std::vector<uint32_t>> preds(G.n_nodes);
    const auto e = I.view->edges(gi);
    for (uint32_t k = 0; k < G.n_edges; ++k) preds[e[2 * k + 1]].push_back(e[2 * k]);

    I.dev->make_current();
    cudaStream_t st = nullptr;  // a private stream: nothing else may join the capture
    cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate(capture)");
    std::vector<CUgraphNode> captured(G.n_nodes, nullptr);
    cudaGraph_t graph = nullptr;
    auto cleanup = [&] {
        if (graph) cudaGraphDestroy(graph);
        cudaStreamDestroy(st);
    };
    try {
        cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
        for (uint32_t n = 0; n < G.n_nodes; ++n) {
            std::vector<cudaGraphNode_t> deps;
            for (uint32_t p : preds[n]) deps.push_back(reinterpret_cast<cudaGraphNode_t>(captured[p]));
            cuda_check(cudaStreamUpdateCaptureDependencies(st, deps.data(), deps.size(),
                                                           cudaStreamSetCaptureDependencies),
                       "cudaStreamUpdateCaptureDependencies");
            fdt_node d;
            std::memcpy(&d, img + 48ull * n, sizeof d);
            const uint8_t* blob = pool + d.blob_off;
            if (d.type == 0) {
                const auto& K = I.resolve(d.kernel, n);
                size_t size = K.arg_buffer_size;
                void* extra[5] = {CU_LAUNCH_PARAM_BUFFER_POINTER, const_cast<uint8_t*>(blob),
                                  CU_LAUNCH_PARAM_BUFFER_SIZE, &size, CU_LAUNCH_PARAM_END};
                // the launch attributes the template build applies (build_graph_for)
                const fdt_node_attrs& a = I.view->node_attrs(gi, n);
                CUlaunchAttribute attrs[2];
                unsigned na = 0;
                const uint32_t csize = a.cluster[0] * a.cluster[1] * a.cluster[2];
                if (csize > 1 && csize <= 8 && d.grid[0] % a.cluster[0] == 0 && d.grid[1] % a.cluster[1] == 0 &&
                    d.grid[2] % a.cluster[2] == 0) {
                    attrs[na].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
                    attrs[na].value.clusterDim.x = a.cluster[0];
                    attrs[na].value.clusterDim.y = a.cluster[1];
                    attrs[na].value.clusterDim.z = a.cluster[2];
                    ++na;
                }
                if (a.sched_policy > 0 && a.sched_policy <= 2) {
                    attrs[na].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_SCHEDULING_POLICY_PREFERENCE;
                    attrs[na].value.clusterSchedulingPolicyPreference =
                        static_cast<CUclusterSchedulingPolicy>(a.sched_policy);
                    ++na;
                }
                CUlaunchConfig cfg{};
                cfg.gridDimX = d.grid[0], cfg.gridDimY = d.grid[1], cfg.gridDimZ = d.grid[2];
                cfg.blockDimX = d.block[0], cfg.blockDimY = d.block[1], cfg.blockDimZ = d.block[2];
                cfg.sharedMemBytes = d.shmem;
                cfg.hStream = st;
                cfg.attrs = na ? attrs : nullptr;
                cfg.numAttrs = na;
                cu_check(api.cuLaunchKernelEx(&cfg, I.ctx->function(K), nullptr, extra), "cuLaunchKernelEx(capture)");
            } else if (d.type == 1) {
                cuda_check(cudaMemcpyAsync(reinterpret_cast<void*>(rd64(blob + 8)),
                                           reinterpret_cast<const void*>(rd64(blob)), rd64(blob + 16),
                                           cudaMemcpyDeviceToDevice, st),
                           "cudaMemcpyAsync(capture)");
            } else if (d.type == 2) {
                const uint64_t value = rd64(blob + 8), len = rd64(blob + 16);
                if (value <= 0xFF)
                    cu_check(api.cuMemsetD8Async(rd64(blob), static_cast<unsigned char>(value), len, st),
                             "cuMemsetD8Async(capture)");
                else
                    cu_check(api.cuMemsetD32Async(rd64(blob), static_cast<unsigned int>(value), len / 4, st),
                             "cuMemsetD32Async(capture)");
            } else {  // no stream operation makes an empty node: add it to the capture graph
                cudaStreamCaptureStatus status;
                cudaGraph_t cg = nullptr;
                cuda_check(cudaStreamGetCaptureInfo(st, &status, nullptr, &cg), "cudaStreamGetCaptureInfo");
                cudaGraphNode_t empty = nullptr;
                cuda_check(cudaGraphAddEmptyNode(&empty, cg, deps.data(), deps.size()), "cudaGraphAddEmptyNode");
                cuda_check(cudaStreamUpdateCaptureDependencies(st, &empty, 1, cudaStreamSetCaptureDependencies),
                           "cudaStreamUpdateCaptureDependencies");
            }
            // the node just captured is the stream's whole dependency set now
            cudaStreamCaptureStatus status;
            const cudaGraphNode_t* now = nullptr;
            size_t n_now = 0;
            cuda_check(cudaStreamGetCaptureInfo(st, &status, nullptr, nullptr, &now, &n_now),
                       "cudaStreamGetCaptureInfo");
            require(status == cudaStreamCaptureStatusActive && n_now == 1, Errc::cuda_error,
                    "capture of node " + std::to_string(n) + " did not yield exactly one graph node");
            captured[n] = reinterpret_cast<CUgraphNode>(now[0]);
        }
        cuda_check(cudaStreamEndCapture(st, &graph), "cudaStreamEndCapture");
        CapturedGraph g = extract_graph(*I.ctx, reinterpret_cast<CUgraph>(graph), batch, captured);
        cleanup();
        return g;
    } catch (...) {
        if (!graph) {
            cudaGraph_t partial = nullptr;
            cudaStreamEndCapture(st, &partial);  // leave capture mode before unwinding
            if (partial) cudaGraphDestroy(partial);
            cudaGetLastError();
        }
        cleanup();
        throw;
    }
}

// GPU-side SAVE to an archive (reference SAVE pipeline.cpp:249-405).
// Every batch's graph is stream-captured on the device and extracted from the
// driver (capture_graph); the interception record supplies the launch
// attributes each kernel was launched with (the extraction cannot read back
// the ones the hardware does not carry, capture.hpp). The stub layer then
// lowers the rank-specific comm nodes back to stubs with the SAVE-time
// placeholders (the inverse of apply_rank_patches, rank_forge.cpp:132-152:
// kernel -> stub ref, rank bytes -> 0, world bytes -> the table's
// world_placeholder), so one capture from ANY rank yields the rank-agnostic
// archive. Grouping (topology_key + group_graphs, templater.cpp:18-52),
// serialize_graphs (graph_model.cpp:244-269), the catalog of the restored
// binaries (binary_catalog.cpp:108-183), the memory log and the manifest follow
// the reference layout; templates.fdt is packed from the new graphs.bin.
SaveResult ServingContext::save_captured(const fs::path& out) {
    Impl& I = *impl_;
    require(I.t.relocation_delta == 0, Errc::invalid_argument,
            "save_captured: the region was relocated; capture from a LOAD at the captured base");
    require(I.view->header().n_values == 0, Errc::invalid_argument,
            "save_captured: the archive carries comm slots whose SAVE-time values are unknown");
    require(!fs::exists(out) || fs::is_empty(out), Errc::invalid_argument,
            "save_captured: " + out.string() + " exists and is not empty");
    const PatchTable patches = parse_patch_table(I.file_host("patch.bin"));
    std::vector<CapturedGraph> graphs;
    for (uint32_t b : I.labels) {
        CapturedGraph g = capture_graph(b);
        const uint32_t m = I.member_for(b);
        const uint32_t gi = I.view->member(m).group;
        for (uint32_t n = 0; n < g.nodes.size(); ++n) {
            if (g.nodes[n].type != NodeType::Kernel) continue;
            const fdt_node_attrs& a = I.view->node_attrs(gi, n);  // what the launch asked for
            g.nodes[n].attrs.cluster_dim = {a.cluster[0], a.cluster[1], a.cluster[2]};
            g.nodes[n].attrs.cluster_scheduling_policy_preference = a.sched_policy;
            g.nodes[n].attrs.mem_sync_domain_map_default = a.sync_default;
            g.nodes[n].attrs.mem_sync_domain_map_remote = a.sync_remote;
            g.nodes[n].attrs.attr_query_available = a.attr_query != 0;
        }
        auto pit = patches.per_graph.find(b);
        if (pit != patches.per_graph.end()) {
            for (const CommPatchEntry& e : pit->second) {
                require(e.node_id < g.nodes.size() && g.nodes[e.node_id].type == NodeType::Kernel,
                        Errc::archive_corruption, "patch entry references a non-kernel node");
                auto& k = g.nodes[e.node_id].kernel_params();
                require(k.kernel == KernelRef{I.manifest.comm_real_hash, e.real_name}, Errc::unpatchable_comm,
                        "node " + std::to_string(e.node_id) + " of batch " + std::to_string(b) +
                            " is not the real comm kernel its patch entry names");
                k.kernel = e.stub;
                for (uint32_t off : e.rank_offsets) std::memset(k.arg_buffer.data() + off, 0, 8);
                for (uint32_t off : e.world_offsets)
                    std::memcpy(k.arg_buffer.data() + off, &patches.world_placeholder, 8);
            }
        }
        graphs.push_back(std::move(g));
    }
    GroupingManifest grouping = group_graphs(graphs);
    const std::vector<uint8_t> graphs_bin = serialize_graphs(graphs);
    attach_locators(grouping, parse_graph_locators(graphs_bin));

    ArchivePaths paths{out};
    fs::create_directories(paths.binaries());
    Manifest m = I.manifest;
    m.grouping = std::move(grouping);
    m.file_digests.clear();
    auto put = [&](const std::string& rel, std::span<const uint8_t> bytes) {
        spit(out / rel, std::vector<uint8_t>(bytes.begin(), bytes.end()));
        m.file_digests[rel] = crc64(bytes);
    };
    put("graphs.bin", graphs_bin);
    put("memlayout.bin", I.file_host("memlayout.bin"));
    put("catalog.bin", serialize_catalog(I.catalog));
    put("patch.bin", I.file_host("patch.bin"));
    for (const auto& [hash, rec] : I.catalog.binaries) {
        (void)rec;
        for (const std::string& rel : {"binaries/" + hex16(hash) + ".bin", "binaries/" + hex16(hash) + ".sm_100a.cubin"}) {
            if (I.staged->has(rel)) put(rel, I.file_host(rel));
            else if (fs::exists(I.root / rel)) put(rel, slurp(I.root / rel));
        }
    }
    spit(paths.manifest(), serialize_manifest(m));
    pack_archive_store(out, I.opts.prepare_lanes);

    SaveResult res;
    res.archive_dir = out;
    const auto mt = slurp(paths.manifest());
    res.manifest = parse_manifest(std::string(mt.begin(), mt.end()));
    return res;
}

uint64_t ServingContext::naive_rebuild_all() {
    Impl& I = *impl_;
    const DriverApi& api = driver();
    uint64_t calls = 0;
    for (uint32_t m = 0; m < I.view->n_members(); ++m) {
        const uint32_t gi = I.view->member(m).group;
        CUgraph g = nullptr;
        CUgraphExec x = nullptr;
        std::vector<CUgraphNode> nodes;
        calls += I.build_graph_for(gi, m, g, nodes);
        cu_check(api.cuGraphInstantiate(&x, g, 0), "cuGraphInstantiate");
        ++calls;
        cu_check(api.cuGraphLaunch(x, I.dev->stream()), "cuGraphLaunch");
        I.dev->sync();
        api.cuGraphExecDestroy(x);
        api.cuGraphDestroy(g);
    }
    return calls;
}

void ServingContext::exec_update(uint32_t batch_in_group, const CapturedGraph& donor) {
    Impl& I = *impl_;
    const uint32_t m = I.member_for(batch_in_group);
    const uint32_t gi = I.view->member(m).group;
    const fdt_group& G = I.view->group(gi);
    donor.validate();
    for (const auto& n : donor.nodes) {
        if (n.type != NodeType::Kernel) continue;
        const auto& k = n.kernel_params();
        const auto* K = I.ctx->find_kernel(k.kernel.binary_hash, k.kernel.name);
        require(K != nullptr, Errc::unresolved_kernel,
                "node " + std::to_string(n.id) + " references " + k.kernel.describe());
        require(k.arg_buffer.size() >= K->arg_buffer_size, Errc::invalid_argument,
                "exec_update: argument buffer smaller than '" + K->name + "' declares");
    }
    const TopologyKey want{Digest128{G.key_hi, G.key_lo}};
    const TopologyKey got = topology_key(donor);
    require(got == want, Errc::topology_mismatch,
            "donor topology " + got.hex() + " does not match exec topology " + want.hex());
    // donor parameters are applied node by node; the exec no longer holds a member
    const DriverApi& api = driver();
    I.dev->make_current();
    Impl::Group& grp = I.exec_of(gi);
    for (uint32_t n = 0; n < G.n_nodes; ++n) {
        const GraphNode& node = donor.nodes[n];
        if (node.type == NodeType::Kernel) {
            const auto& k = node.kernel_params();
            const auto* K = I.ctx->find_kernel(k.kernel.binary_hash, k.kernel.name);
            fdt_node d{};
            d.grid[0] = k.grid.x, d.grid[1] = k.grid.y, d.grid[2] = k.grid.z;
            d.block[0] = k.block.x, d.block[1] = k.block.y, d.block[2] = k.block.z;
            d.shmem = k.shared_mem_bytes;
            CUDA_KERNEL_NODE_PARAMS p;
            void* extra[5];
            size_t size;
            I.kernel_params(d, k.arg_buffer.data(), *K, p, extra, &size);
            cu_check(api.cuGraphExecKernelNodeSetParams(grp.exec, grp.nodes[n], &p),
                     "cuGraphExecKernelNodeSetParams");
        } else if (node.type == NodeType::Memcpy) {
            const auto& c = std::get<MemcpyParams>(node.params);
            const uint64_t raw[3] = {c.src, c.dst, c.length};
            const CUDA_MEMCPY3D cp = I.memcpy_params(reinterpret_cast<const uint8_t*>(raw));
            cu_check(api.cuGraphExecMemcpyNodeSetParams(grp.exec, grp.nodes[n], &cp, I.cu_ctx),
                     "cuGraphExecMemcpyNodeSetParams");
        } else if (node.type == NodeType::Memset) {
            const auto& s = std::get<MemsetParams>(node.params);
            const uint64_t raw[3] = {s.dst, s.value, s.length};
            const CUDA_MEMSET_NODE_PARAMS sp = I.memset_params(reinterpret_cast<const uint8_t*>(raw));
            cu_check(api.cuGraphExecMemsetNodeSetParams(grp.exec, grp.nodes[n], &sp, I.cu_ctx),
                     "cuGraphExecMemsetNodeSetParams");
        }
    }
    if (I.opts.device_updates && !grp.serve_nodes.empty()) {
        cu_check(api.cuGraphUpload(grp.exec, I.dev->stream()), "cuGraphUpload");
        for (auto& r : grp.memops) r = {~0ull, ~0ull, ~0ull};  // unknown: the next serve re-applies memops
    }
    grp.applied = kNoMember;
    grp.bound = gi;
    ++I.lane_acquisitions;
    I.ctx->c_update.fetch_add(1);
    I.ctx->c_update_touched.fetch_add(G.n_nodes);
}

}  // namespace foundry
