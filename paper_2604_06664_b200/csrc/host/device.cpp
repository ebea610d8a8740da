// Device runtime: streams, HBM/pinned buffers, kernel launches (see device.hpp).
#include "foundry/device.hpp"

#include <cstring>
#include <mutex>
#include <string>

#include <cuda_runtime.h>

#include "../kernels/fdy_kernels.h"
#include "foundry/hash.hpp"
#include "foundry/staging.hpp"

namespace foundry {

void cuda_check(int err, const char* what) {
    if (err == cudaSuccess) return;
    const auto e = static_cast<cudaError_t>(err);
    const bool no_device = e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ||
                           e == cudaErrorInitializationError;
    raise(no_device ? Errc::device_unavailable : Errc::cuda_error,
          std::string(what) + " failed: " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

int cuda_device_count() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();  // clear the sticky-free error state
        return 0;
    }
    return n;
}

bool cuda_available() { return cuda_device_count() > 0; }

namespace {
std::once_flag g_const_once[64];
std::once_flag g_pool_once[64];
}

Device::Device(int ordinal) : ordinal_(ordinal) {
    const int n = cuda_device_count();
    require(n > 0, Errc::device_unavailable, "no CUDA device is visible (the B200 path has no CPU fallback)");
    require(ordinal >= 0 && ordinal < n, Errc::invalid_argument,
            "device ordinal " + std::to_string(ordinal) + " out of range (" + std::to_string(n) + " visible)");
    cuda_check(cudaSetDevice(ordinal_), "cudaSetDevice");
    cuda_check(cudaFree(nullptr), "cudaFree(0) context init");
    cuda_check(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, ordinal_),
               "cudaDeviceGetAttribute(SM count)");
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&side_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    // per-device constant table of the CRC kernel: x^(2^k) mod P
    std::call_once(g_const_once[ordinal_ & 63], [] {
        cuda_check(fdy_crc64_set_constants(crc64_x2k_table()), "CRC constant upload");
    });
    // the default pool keeps what it is given back (see alloc())
    std::call_once(g_pool_once[ordinal_ & 63], [this] {
        cudaMemPool_t pool;
        cuda_check(cudaDeviceGetDefaultMemPool(&pool, ordinal_), "cudaDeviceGetDefaultMemPool");
        uint64_t keep = UINT64_MAX;
        cuda_check(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep),
                   "cudaMemPoolSetAttribute(release threshold)");
    });
}

Device::~Device() {
    cudaSetDevice(ordinal_);
    if (stream_) cudaStreamDestroy(stream_);
    if (copy_stream_) cudaStreamDestroy(copy_stream_);
    if (side_stream_) cudaStreamDestroy(side_stream_);
}

void Device::make_current() const { cuda_check(cudaSetDevice(ordinal_), "cudaSetDevice"); }

void Device::sync() const {
    cuda_check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
    cuda_check(cudaStreamSynchronize(copy_stream_), "cudaStreamSynchronize(copy)");
    cuda_check(cudaStreamSynchronize(side_stream_), "cudaStreamSynchronize(side)");
}

void* Device::alloc(size_t bytes, bool shareable) {
    make_current();
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    if (shareable)
        cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    else
        cuda_check(cudaMallocAsync(&p, bytes, stream_), "cudaMallocAsync");
    return p;
}

void Device::release(void* p, bool shareable) {
    if (!p) return;
    cudaSetDevice(ordinal_);
    if (shareable)
        cudaFree(p);
    else
        cudaFreeAsync(p, stream_);
}

void* Device::alloc_host_pinned(size_t bytes) {
    make_current();
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    cuda_check(cudaHostAlloc(&p, bytes, cudaHostAllocPortable), "cudaHostAlloc");
    return p;
}

void Device::release_host_pinned(void* p) {
    if (p) cudaFreeHost(p);
}

DeviceBuffer::DeviceBuffer(Device& dev, size_t bytes, bool shareable)
    : dev_(&dev), p_(static_cast<unsigned char*>(dev.alloc(bytes, shareable))), n_(bytes),
      shareable_(shareable) {}

DeviceBuffer::~DeviceBuffer() {
    if (dev_) dev_->release(p_, shareable_);
}

DeviceBuffer& DeviceBuffer::operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
        if (dev_) dev_->release(p_, shareable_);
        dev_ = o.dev_;
        p_ = o.p_;
        n_ = o.n_;
        shareable_ = o.shareable_;
        o.dev_ = nullptr;
        o.p_ = nullptr;
        o.n_ = 0;
    }
    return *this;
}

PinnedBuffer::PinnedBuffer(Device& dev, size_t bytes)
    : dev_(&dev), p_(static_cast<unsigned char*>(dev.alloc_host_pinned(bytes))), n_(bytes) {}

PinnedBuffer::~PinnedBuffer() {
    if (dev_) dev_->release_host_pinned(p_);
}

PinnedBuffer& PinnedBuffer::operator=(PinnedBuffer&& o) noexcept {
    if (this != &o) {
        if (dev_) dev_->release_host_pinned(p_);
        dev_ = o.dev_;
        p_ = o.p_;
        n_ = o.n_;
        o.dev_ = nullptr;
        o.p_ = nullptr;
        o.n_ = 0;
    }
    return *this;
}

// ------------------------------------------------------------------ stores

DeviceStore adopt_store(Device& dev, const unsigned char* d_blob, size_t bytes, const fdt_header& h) {
    require(bytes >= sizeof(fdt_header) && std::memcmp(h.magic, "FNDT", 4) == 0,
            Errc::archive_corruption, "template store: bad magic, expected 'FNDT'");
    require(h.version == FDT_VERSION, Errc::archive_corruption,
            "template store: unsupported version " + std::to_string(h.version));
    for (int i = 0; i < FDT_NSEC; ++i)
        require(h.sec[i].offset <= bytes && h.sec[i].bytes <= bytes - h.sec[i].offset,
                Errc::archive_corruption, "template store: section overruns the blob");
    require(h.tile_chunks == FDT_TILE_CHUNKS, Errc::archive_corruption,
            "template store: tile size " + std::to_string(h.tile_chunks) + " unsupported");
    DeviceStore s;
    s.dev = &dev;
    s.data = d_blob;
    s.bytes = bytes;
    s.header = h;
    if (h.sec[FDT_SEC_TIMAGES].bytes) s.rtimages = DeviceBuffer(dev, h.sec[FDT_SEC_TIMAGES].bytes);
    require(h.n_plain_tiles <= h.n_tiles, Errc::archive_corruption,
            "template store: more relocation-free tiles than tiles");
    return s;
}

DeviceStore upload_store(Device& dev, const void* host_blob, size_t bytes) {
    require(bytes >= sizeof(fdt_header), Errc::archive_corruption, "template store: truncated input");
    fdt_header h;
    std::memcpy(&h, host_blob, sizeof h);
    DeviceBuffer buf(dev, bytes, /*shareable=*/true);  // fdy_store_export may hand it to peers
    cuda_check(cudaMemcpyAsync(buf.data(), host_blob, bytes, cudaMemcpyHostToDevice, dev.stream()),
               "cudaMemcpyAsync(store H2D)");
    DeviceStore s = adopt_store(dev, buf.data(), bytes, h);
    s.blob = std::move(buf);
    return s;
}

void check_store_sources(const fdt_header& h, const Manifest& manifest) {
    const auto slots = manifest.file_digests.find("comm_slots.bin");
    require(h.source_graphs_crc == manifest.file_digests.at("graphs.bin") &&
                h.source_patch_crc == manifest.file_digests.at("patch.bin"),
            Errc::archive_corruption, "template store was packed from a different graphs.bin/patch.bin");
    require(h.source_slots_crc == (slots == manifest.file_digests.end() ? 0ull : slots->second),
            Errc::archive_corruption, "template store was packed from a different comm_slots.bin");
    if (h.n_rank_ops > 0)
        require(manifest.comm_real_hash != 0, Errc::unresolved_kernel,
                "archive carries comm patches but no real comm binary");
}

void launch_materialize(Device& dev, const DeviceStore& store, const MaterializeRequest& req,
                        unsigned char* out, MaterializeTiming* timing, int grid_override) {
    const fdt_header& h = store.header;
    require(req.world >= 1 && req.rank < req.world, Errc::invalid_argument,
            "rank " + std::to_string(req.rank) + " is outside world size " + std::to_string(req.world));
    require(req.values.size() >= h.n_values, Errc::invalid_argument,
            "the archive's comm slots read " + std::to_string(h.n_values) + " per-rank values, " +
                std::to_string(req.values.size()) + " given (LoadOptions::comm_values)");
    dev.make_current();
    const uint64_t* d_values = nullptr;
    if (!req.values.empty()) {
        const size_t vb = req.values.size() * sizeof(uint64_t);
        if (store.values.size() < vb) store.values = DeviceBuffer(dev, vb);
        cuda_check(cudaMemcpyAsync(store.values.data(), req.values.data(), vb, cudaMemcpyHostToDevice,
                                   dev.stream()),
                   "cudaMemcpyAsync(value table)");
        d_values = reinterpret_cast<const uint64_t*>(store.values.data());
    }
    FdyMaterializeArgs a{};
    const unsigned char* b = store.data;
    a.store = b;
    a.out = out;
    a.rtimg = store.rtimages.data();
    a.tiles = reinterpret_cast<const fdt_tile*>(b + h.sec[FDT_SEC_TILES].offset);
    a.cmeta = b + h.sec[FDT_SEC_CMETA].offset;
    a.didx = reinterpret_cast<const uint16_t*>(b + h.sec[FDT_SEC_DIDX].offset);
    a.ddata = reinterpret_cast<const uint64_t*>(b + h.sec[FDT_SEC_DDATA].offset);
    a.rops = reinterpret_cast<const fdt_rank_op*>(b + h.sec[FDT_SEC_ROPS].offset);
    a.values = d_values;
    a.n_values = d_values ? static_cast<uint32_t>(req.values.size()) : 0u;
    a.timage_base = h.sec[FDT_SEC_TIMAGES].offset;
    a.timage_bytes = h.sec[FDT_SEC_TIMAGES].bytes;
    a.old_base = h.old_base;
    a.span = h.final_offset;
    a.delta = req.new_base ? req.new_base - h.old_base : 0;
    a.rank = req.rank;
    a.world = req.world;
    a.n_tiles = h.n_tiles;
    a.n_plain = h.n_plain_tiles;  // the packer stored the relocation-free tiles first
    // the kernel reads template chunks at tsrc + tile.src_off (a store offset)
    a.tsrc = a.delta && a.rtimg ? reinterpret_cast<const unsigned char*>(
                                      reinterpret_cast<uintptr_t>(a.rtimg) - a.timage_base)
                                : b;

    int per_sm = 0;
    cuda_check(fdy_materialize_occupancy(&per_sm), "materialize occupancy query");
    int grid = grid_override > 0 ? grid_override : dev.sm_count() * std::max(per_sm, 1);
    grid = std::max(1, std::min<int>(grid, static_cast<int>(h.n_tiles)));

    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing) {
        cuda_check(cudaEventCreate(&e0), "cudaEventCreate");
        cuda_check(cudaEventCreate(&e1), "cudaEventCreate");
        // hold the stream while the launches are submitted: the events then
        // bracket device time only (the host's launch latency is not in it)
        if (timing->gate) cuda_check(fdy_launch_gate(dev.stream(), 50000), "gate kernel launch");
        cuda_check(cudaEventRecord(e0, dev.stream()), "cudaEventRecord");
    }
    cudaEvent_t em = nullptr;
    if (timing && timing->split) {
        cuda_check(cudaEventCreate(&em), "cudaEventCreate");
        cuda_check(fdy_launch_materialize_split(&a, grid, dev.stream(), em), "materialize kernel launch");
    } else {
        cuda_check(fdy_launch_materialize(&a, grid, dev.stream()), "materialize kernel launch");
    }
    if (timing) {
        cuda_check(cudaEventRecord(e1, dev.stream()), "cudaEventRecord");
        cuda_check(cudaEventSynchronize(e1), "cudaEventSynchronize");
        cuda_check(cudaEventElapsedTime(&timing->kernel_ms, e0, e1), "cudaEventElapsedTime");
        if (em) {
            cuda_check(cudaEventElapsedTime(&timing->reloc_ms, e0, em), "cudaEventElapsedTime");
            cuda_check(cudaEventElapsedTime(&timing->member_ms, em, e1), "cudaEventElapsedTime");
            cudaEventDestroy(em);
        }
        timing->grid = grid;
        timing->blocks_per_sm = per_sm;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
}

// ------------------------------------------------------------------ CRC

std::vector<uint64_t> crc64_device(Device& dev, const unsigned char* d_base,
                                   std::span<const Segment> segments, float* kernel_ms) {
    dev.make_current();
    std::vector<FdyCrcBlock> blocks;
    std::vector<uint32_t> first(segments.size()), count(segments.size());
    for (size_t s = 0; s < segments.size(); ++s) {
        first[s] = static_cast<uint32_t>(blocks.size());
        for (uint64_t off = 0; off < segments[s].length; off += kCrcBlockBytes) {
            FdyCrcBlock b;
            b.segment = static_cast<uint32_t>(s);
            b.length = static_cast<uint32_t>(std::min<uint64_t>(kCrcBlockBytes, segments[s].length - off));
            b.offset = segments[s].offset + off;
            blocks.push_back(b);
        }
        count[s] = static_cast<uint32_t>(blocks.size()) - first[s];
        require(count[s] <= kCrcMaxSegmentBlocks, Errc::invalid_argument, "CRC segment longer than 64 GiB");
    }
    const size_t nb = blocks.size(), ns = segments.size();
    // one scratch allocation: block table | first | count | crc | len | out
    const size_t bytes = nb * sizeof(FdyCrcBlock) + 2 * ns * 4 + 2 * nb * 8 + ns * 8 + 64;
    DeviceBuffer scratch(dev, bytes);
    unsigned char* p = scratch.data();
    auto* d_blocks = reinterpret_cast<FdyCrcBlock*>(p);
    p += nb * sizeof(FdyCrcBlock);
    auto* d_crc = reinterpret_cast<uint64_t*>(p);
    p += nb * 8;
    auto* d_len = reinterpret_cast<uint64_t*>(p);
    p += nb * 8;
    auto* d_out = reinterpret_cast<uint64_t*>(p);
    p += ns * 8;
    auto* d_first = reinterpret_cast<uint32_t*>(p);
    p += ns * 4;
    auto* d_count = reinterpret_cast<uint32_t*>(p);
    cudaStream_t st = dev.stream();
    if (nb) cuda_check(cudaMemcpyAsync(d_blocks, blocks.data(), nb * sizeof(FdyCrcBlock), cudaMemcpyHostToDevice, st), "H2D crc plan");
    if (ns) {
        cuda_check(cudaMemcpyAsync(d_first, first.data(), ns * 4, cudaMemcpyHostToDevice, st), "H2D crc plan");
        cuda_check(cudaMemcpyAsync(d_count, count.data(), ns * 4, cudaMemcpyHostToDevice, st), "H2D crc plan");
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (kernel_ms) {
        cuda_check(cudaEventCreate(&e0), "cudaEventCreate");
        cuda_check(cudaEventCreate(&e1), "cudaEventCreate");
        cuda_check(cudaEventRecord(e0, st), "cudaEventRecord");
    }
    cuda_check(fdy_launch_crc64(d_base, d_blocks, static_cast<uint32_t>(nb), d_first, d_count,
                                static_cast<uint32_t>(ns), d_crc, d_len, d_out, st),
               "crc64 kernel launch");
    if (kernel_ms) cuda_check(cudaEventRecord(e1, st), "cudaEventRecord");
    std::vector<uint64_t> out(ns);
    if (ns) cuda_check(cudaMemcpyAsync(out.data(), d_out, ns * 8, cudaMemcpyDeviceToHost, st), "D2H crc");
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize(crc)");
    if (kernel_ms) {
        cuda_check(cudaEventElapsedTime(kernel_ms, e0, e1), "cudaEventElapsedTime");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    return out;
}

CrcJob::~CrcJob() {
    // side-stream work may still read the scratch / write the pinned digests
    // (an error path between launch and join): let it finish before they go
    if (dev_ && on_ && on_ != dev_->stream()) cudaStreamSynchronize(on_);
    if (fork_) cudaEventDestroy(fork_);
    if (done_) cudaEventDestroy(done_);
}

void CrcJob::launch(Device& dev, const unsigned char* d_base, std::span<const Segment> segments,
                    cudaStream_t on) {
    dev.make_current();
    if (dev_ && on_ && on_ != dev_->stream()) cuda_check(cudaStreamSynchronize(on_), "cudaStreamSynchronize(crc)");
    dev_ = &dev;
    on_ = on ? on : dev.stream();
    ns_ = segments.size();
    size_t nb = 0;
    for (const Segment& g : segments) nb += (g.length + kCrcBlockBytes - 1) / kCrcBlockBytes;
    // plan in pinned memory (one async copy): block table | first | count
    const size_t plan_bytes = nb * sizeof(FdyCrcBlock) + 8 * ns_;
    plan_ = PinnedLease(dev, std::max<size_t>(plan_bytes, 16));
    out_ = PinnedLease(dev, std::max<size_t>(8 * ns_, 16));
    auto* blocks = reinterpret_cast<FdyCrcBlock*>(plan_.data());
    auto* first = reinterpret_cast<uint32_t*>(plan_.data() + nb * sizeof(FdyCrcBlock));
    auto* count = first + ns_;
    uint32_t b = 0;
    for (size_t s = 0; s < ns_; ++s) {
        first[s] = b;
        for (uint64_t off = 0; off < segments[s].length; off += kCrcBlockBytes) {
            FdyCrcBlock& k = blocks[b++];
            k = FdyCrcBlock{};
            k.segment = static_cast<uint32_t>(s);
            k.length = static_cast<uint32_t>(std::min<uint64_t>(kCrcBlockBytes, segments[s].length - off));
            k.offset = segments[s].offset + off;
        }
        count[s] = b - first[s];
        require(count[s] <= kCrcMaxSegmentBlocks, Errc::invalid_argument, "CRC segment longer than 64 GiB");
    }
    // device scratch: plan | crc | len | out
    const size_t dev_bytes = (plan_bytes + 15) / 16 * 16 + 2 * nb * 8 + ns_ * 8 + 64;
    scratch_ = DeviceBuffer(dev, dev_bytes);
    unsigned char* p = scratch_.data();
    auto* d_blocks = reinterpret_cast<FdyCrcBlock*>(p);
    auto* d_first = reinterpret_cast<uint32_t*>(p + nb * sizeof(FdyCrcBlock));
    auto* d_count = d_first + ns_;
    p += (plan_bytes + 15) / 16 * 16;
    auto* d_crc = reinterpret_cast<uint64_t*>(p);
    auto* d_len = d_crc + nb;
    auto* d_out = d_len + nb;
    cudaStream_t st = on_;
    if (st != dev.stream()) {  // the scratch (stream-ordered on dev.stream()) and the input first
        if (!fork_) cuda_check(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventRecord(fork_, dev.stream()), "cudaEventRecord(crc fork)");
        cuda_check(cudaStreamWaitEvent(st, fork_, 0), "cudaStreamWaitEvent(crc fork)");
    }
    if (plan_bytes)
        cuda_check(cudaMemcpyAsync(scratch_.data(), plan_.data(), plan_bytes, cudaMemcpyHostToDevice, st),
                   "H2D crc plan");
    cuda_check(fdy_launch_crc64(d_base, d_blocks, static_cast<uint32_t>(nb), d_first, d_count,
                                static_cast<uint32_t>(ns_), d_crc, d_len, d_out, st),
               "crc64 kernel launch");
    if (ns_) cuda_check(cudaMemcpyAsync(out_.data(), d_out, ns_ * 8, cudaMemcpyDeviceToHost, st), "D2H crc");
    if (st != dev.stream()) {
        if (!done_) cuda_check(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventRecord(done_, st), "cudaEventRecord(crc done)");
    }
}

void CrcJob::join(cudaStream_t st) {
    if (dev_ && on_ != st && done_) cuda_check(cudaStreamWaitEvent(st, done_, 0), "cudaStreamWaitEvent(crc join)");
}

std::span<const uint64_t> CrcJob::wait() {
    if (dev_) cuda_check(cudaStreamSynchronize(on_), "cudaStreamSynchronize(crc)");
    return digests();
}

}  // namespace foundry
