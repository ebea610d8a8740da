// Archive staging with overlapped reads + DMA, pinned pool, GPU integrity.
#include "foundry/staging.hpp"
#include "foundry/device_pack.hpp"

#include <fcntl.h>
#include <sys/resource.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <future>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <optional>
#include <thread>

#include <cuda_runtime.h>

#include "foundry/bytes.hpp"
#include "foundry/hash.hpp"
#include "foundry/parallel.hpp"
#include "../kernels/fdy_kernels.h"

namespace foundry {

namespace fs = std::filesystem;

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

constexpr size_t kAlign = 256;

// FOUNDRY_DEBUG=1: timeline of the end-to-end path on stderr (diagnostics)
void trace_point(const char* what, Clock::time_point t0) {
    static const bool on = std::getenv("FOUNDRY_DEBUG") != nullptr;
    if (on) std::fprintf(stderr, "[foundry] %8.3f ms  %s\n", ms_since(t0), what);
}
// 2 MiB: one pread of it takes ~1 ms on a lane, so the store (read first)
// is spread over every lane and the last pieces balance across lanes
constexpr size_t kPiece = 2ull << 20;

struct PoolEntry {
    int device;
    unsigned char* p;
    size_t cap;
};

std::mutex g_pool_mu;
std::vector<PoolEntry> g_pool;  // free pinned buffers

void read_range(const fs::path& p, uint8_t* dst, uint64_t off, uint64_t len) {
    const int fd = ::open(p.c_str(), O_RDONLY | O_CLOEXEC);
    require(fd >= 0, Errc::archive_corruption, "cannot open " + p.string());
    uint64_t done = 0;
    while (done < len) {
        const ssize_t n = ::pread(fd, dst + done, len - done, static_cast<off_t>(off + done));
        if (n <= 0) {
            ::close(fd);
            raise(Errc::archive_corruption, "short read on " + p.string());
        }
        done += static_cast<uint64_t>(n);
    }
    ::close(fd);
}

}  // namespace

// ------------------------------------------------------------------ pinned pool

PinnedLease::PinnedLease(Device& dev, size_t bytes) : n_(bytes), device_(dev.ordinal()) {
    {
        std::lock_guard lock(g_pool_mu);
        size_t best = g_pool.size();
        for (size_t i = 0; i < g_pool.size(); ++i)
            if (g_pool[i].cap >= bytes && (best == g_pool.size() || g_pool[i].cap < g_pool[best].cap))
                best = i;
        if (best < g_pool.size()) {
            p_ = g_pool[best].p;
            cap_ = g_pool[best].cap;
            g_pool.erase(g_pool.begin() + static_cast<long>(best));
            return;
        }
    }
    cap_ = std::max<size_t>(bytes, 1 << 20);
    p_ = static_cast<unsigned char*>(dev.alloc_host_pinned(cap_));
}

PinnedLease::~PinnedLease() {
    if (!p_) return;
    std::lock_guard lock(g_pool_mu);
    g_pool.push_back({device_, p_, cap_});
}

PinnedLease& PinnedLease::operator=(PinnedLease&& o) noexcept {
    if (this != &o) {
        if (p_) {
            std::lock_guard lock(g_pool_mu);
            g_pool.push_back({device_, p_, cap_});
        }
        p_ = o.p_;
        n_ = o.n_;
        cap_ = o.cap_;
        device_ = o.device_;
        o.p_ = nullptr;
        o.n_ = o.cap_ = 0;
    }
    return *this;
}

// ------------------------------------------------------------------ pageable pool

namespace {
std::mutex g_pageable_mu;
std::vector<std::pair<unsigned char*, size_t>> g_pageable;
}  // namespace

PageableLease::PageableLease(size_t bytes) {
    {
        std::lock_guard lock(g_pageable_mu);
        size_t best = g_pageable.size();
        for (size_t i = 0; i < g_pageable.size(); ++i)
            if (g_pageable[i].second >= bytes && (best == g_pageable.size() || g_pageable[i].second < g_pageable[best].second))
                best = i;
        if (best < g_pageable.size()) {
            p_ = g_pageable[best].first;
            cap_ = g_pageable[best].second;
            g_pageable.erase(g_pageable.begin() + static_cast<long>(best));
            return;
        }
    }
    cap_ = std::max<size_t>(bytes, 1 << 20);
    p_ = new unsigned char[cap_];
}

PageableLease::~PageableLease() {
    if (!p_) return;
    std::lock_guard lock(g_pageable_mu);
    g_pageable.push_back({p_, cap_});
}

PageableLease& PageableLease::operator=(PageableLease&& o) noexcept {
    if (this != &o) {
        if (p_) {
            std::lock_guard lock(g_pageable_mu);
            g_pageable.push_back({p_, cap_});
        }
        p_ = o.p_;
        cap_ = o.cap_;
        o.p_ = nullptr;
        o.cap_ = 0;
    }
    return *this;
}

// ------------------------------------------------------------------ staging

namespace {
constexpr size_t kScratch = 1 << 20;  // hash-only reads: per-lane, stays in cache

// Hash-only read buffers outlive the lanes that use them: a fresh buffer per
// lane per call would page-fault 256 times per MiB inside every LOAD.
std::mutex g_scratch_mu;
std::vector<std::unique_ptr<uint8_t[]>> g_scratch;

struct ScratchLease {
    std::unique_ptr<uint8_t[]> p;
    uint8_t* get() {
        if (!p) {
            {
                std::lock_guard lock(g_scratch_mu);
                if (!g_scratch.empty()) {
                    p = std::move(g_scratch.back());
                    g_scratch.pop_back();
                }
            }
            if (!p) p.reset(new uint8_t[kScratch]);
        }
        return p.get();
    }
    ~ScratchLease() {
        if (!p) return;
        std::lock_guard lock(g_scratch_mu);
        g_scratch.push_back(std::move(p));
    }
};
}  // namespace

struct StagedArchive::Shared {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<uint32_t> pieces_left;  // per segment
    std::vector<uint8_t> ready;         // per segment: every piece read (and queued / CRCed)
    std::vector<cudaEvent_t> done;      // per device segment, recorded after its fold
    std::vector<uint64_t> piece_crc;    // host / hash files
    std::vector<uint64_t> piece_len;
    std::vector<uint64_t> cpu_digest;   // per segment (host / hash files)
    std::exception_ptr error;           // first reader failure
    size_t remaining = 0;               // pieces not yet done
    std::vector<std::thread> lanes;
    Clock::time_point t0;
    double read_ms = 0;
};

namespace {
std::vector<std::string> manifest_files(const Manifest& m) {
    std::vector<std::string> out;
    for (const auto& [rel, digest] : m.file_digests) out.push_back(rel);
    return out;
}
}  // namespace

StagedArchive::StagedArchive(Device& dev, const fs::path& root, const Manifest& manifest,
                             unsigned lanes, StageTimings* t, StagePlan plan)
    : StagedArchive(dev, root, manifest_files(manifest), lanes, t, std::move(plan)) {}

StagedArchive::StagedArchive(Device& dev, const fs::path& root, const std::vector<std::string>& names,
                             unsigned lanes, StageTimings* t, StagePlan plan)
    : dev_(dev), sh_(std::make_unique<Shared>()) {
    sh_->t0 = Clock::now();
    dev.make_current();  // may run on a helper thread (materialize_archive)
    for (const auto& rel : names) {
        std::error_code ec;
        const uint64_t n = fs::file_size(root / rel, ec);
        require(!ec, Errc::archive_corruption, "cannot open " + (root / rel).string());
        StagedFile f;
        f.rel = rel;
        f.length = n;
        f.placement = plan.keep_host && plan.keep_host(rel) ? Placement::host : Placement::hash;
        files_[rel] = f;
    }
    for (const auto& rel : plan.host_first)
        if (files_.count(rel) && files_.at(rel).placement == Placement::host) order_.push_back(&files_.at(rel));
    for (const auto& rel : plan.device)
        if (files_.count(rel) && files_.at(rel).placement != Placement::device) {
            files_.at(rel).placement = Placement::device;
            order_.push_back(&files_.at(rel));
        }
    for (Placement pl : {Placement::host, Placement::hash})
        for (const auto& [rel, f] : files_)
            if (f.placement == pl && std::find(order_.begin(), order_.end(), &f) == order_.end())
                order_.push_back(&f);

    // layout: device + host files in staging memory; device files' CRC plan
    std::vector<FdyCrcBlock> blocks;
    std::vector<uint32_t> seg_first, seg_count;
    uint32_t n_pieces = 0;
    for (size_t i = 0; i < order_.size(); ++i) {
        StagedFile& f = files_.at(order_[i]->rel);
        f.segment = static_cast<uint32_t>(i);
        if (f.placement == Placement::device) {
            f.offset = device_bytes_;
            device_bytes_ += (f.length + kAlign - 1) / kAlign * kAlign;
        } else if (f.placement == Placement::host) {
            f.offset = host_bytes_;
            host_bytes_ += (f.length + kAlign - 1) / kAlign * kAlign;
        }
        if (f.placement == Placement::device) {
            f.dseg = static_cast<uint32_t>(seg_first.size());
            f.first_block = static_cast<uint32_t>(blocks.size());
            for (uint64_t o = 0; o < f.length; o += kCrcBlockBytes)
                blocks.push_back({f.dseg, static_cast<uint32_t>(std::min<uint64_t>(kCrcBlockBytes, f.length - o)),
                                  f.offset + o});
            f.n_blocks = static_cast<uint32_t>(blocks.size()) - f.first_block;
            require(f.n_blocks <= kCrcMaxSegmentBlocks, Errc::invalid_argument, f.rel + ": longer than 64 GiB");
            seg_first.push_back(f.first_block);
            seg_count.push_back(f.n_blocks);
        } else {
            f.first_piece = n_pieces;
            f.n_pieces = static_cast<uint32_t>((f.length + kPiece - 1) / kPiece);
            n_pieces += f.n_pieces;
        }
    }
    const size_t nb = blocks.size(), nd = seg_first.size(), ns = order_.size();
    trace_point("  staging: layout", sh_->t0);
    total_ = device_bytes_ + host_bytes_;
    host_ = PinnedLease(dev, std::max<uint64_t>(device_bytes_, 16));  // only what the DMA reads is pinned
    pageable_ = PageableLease(std::max<uint64_t>(host_bytes_, 16));
    device_ = DeviceBuffer(dev, std::max<uint64_t>(device_bytes_, 16));
    // GPU CRC scratch: block table | first | count | (align 8) crc | len | digests
    const size_t table = nb * sizeof(FdyCrcBlock), plan_bytes = table + 2 * nd * 4;
    crc_ = DeviceBuffer(dev, plan_bytes + 2 * nb * 8 + nd * 8 + 64);
    digests_ = PinnedLease(dev, std::max<size_t>(plan_bytes, nd * 8) + 64);
    std::memcpy(digests_.data(), blocks.data(), table);
    std::memcpy(digests_.data() + table, seg_first.data(), nd * 4);
    std::memcpy(digests_.data() + table + nd * 4, seg_count.data(), nd * 4);
    auto* d_blocks = reinterpret_cast<FdyCrcBlock*>(crc_.data());
    auto* d_first = reinterpret_cast<uint32_t*>(crc_.data() + table);
    auto* d_count = d_first + nd;
    auto* d_crc = reinterpret_cast<uint64_t*>(crc_.data() + (plan_bytes + 7) / 8 * 8);
    auto* d_len = d_crc + nb;
    auto* d_out = d_len + nb;

    dev.make_current();
    cudaStream_t copy = dev.copy_stream();
    cudaStream_t side = dev.side_stream();
    {  // device buffers are stream-ordered on dev.stream(): copies start after the allocations
        cudaEvent_t allocated;
        cuda_check(cudaEventCreateWithFlags(&allocated, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventRecord(allocated, dev.stream()), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(copy, allocated, 0), "cudaStreamWaitEvent");
        cuda_check(cudaStreamWaitEvent(side, allocated, 0), "cudaStreamWaitEvent");
        cudaEventDestroy(allocated);
    }
    if (plan_bytes) {
        cuda_check(cudaMemcpyAsync(crc_.data(), digests_.data(), plan_bytes, cudaMemcpyHostToDevice, copy),
                   "cudaMemcpyAsync(CRC plan H2D)");
        // the plan must land before the digest slots (same pinned buffer) are reused
        cuda_check(cudaStreamSynchronize(copy), "cudaStreamSynchronize(CRC plan)");
    }

    struct Piece {
        const StagedFile* f;
        uint64_t off, len;
        uint32_t slot;  // host / hash: per-piece CRC slot
    };
    auto pieces = std::make_shared<std::vector<Piece>>();
    for (const StagedFile* f : order_)
        for (uint64_t o = 0, k = 0; o < f->length; o += kPiece, ++k)
            pieces->push_back({f, o, std::min<uint64_t>(kPiece, f->length - o), f->first_piece + static_cast<uint32_t>(k)});
    sh_->pieces_left.assign(ns, 0);
    for (const Piece& pc : *pieces) ++sh_->pieces_left[pc.f->segment];
    sh_->ready.assign(ns, 0);
    sh_->cpu_digest.assign(ns, 0);
    sh_->piece_crc.assign(n_pieces, 0);
    sh_->piece_len.assign(n_pieces, 0);
    sh_->done.assign(nd, nullptr);
    for (auto& e : sh_->done) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    sh_->remaining = pieces->size();
    uint64_t* h_digest = reinterpret_cast<uint64_t*>(digests_.data());  // the plan has landed

    Shared* sh = sh_.get();
    // finishes a file whose pieces are all done (called with sh->mu held)
    auto complete = [=](const StagedFile& f) {
        if (f.placement == Placement::device) {
            cuda_check(fdy_launch_crc64_fold(d_first + f.dseg, d_count + f.dseg, 1, d_crc, d_len,
                                             d_out + f.dseg, side),
                       "CRC fold launch");
            cuda_check(cudaMemcpyAsync(h_digest + f.dseg, d_out + f.dseg, 8, cudaMemcpyDeviceToHost, side),
                       "cudaMemcpyAsync(digest D2H)");
            cuda_check(cudaEventRecord(sh->done[f.dseg], side), "cudaEventRecord");
        } else {
            uint64_t c = 0;  // CRC of the empty string
            for (uint32_t k = 0; k < f.n_pieces; ++k)
                c = k ? crc64_combine(c, sh->piece_crc[f.first_piece + k], sh->piece_len[f.first_piece + k])
                      : sh->piece_crc[f.first_piece];
            sh->cpu_digest[f.segment] = c;
        }
        sh->ready[f.segment] = 1;
    };
    for (const StagedFile* f : order_)  // empty files
        if (sh_->pieces_left[f->segment] == 0) complete(*f);

    trace_point("  staging: buffers + CRC plan", sh_->t0);
    auto next = std::make_shared<std::atomic<size_t>>(0);
    unsigned char* hbase = host_.data();
    unsigned char* pbase = pageable_.data();
    unsigned char* dbase = device_.data();
    const int ordinal = dev.ordinal();
    const fs::path dir = root;  // the lanes outlive this constructor
    const int nice = plan.lane_nice;
    auto body = [=]() {
        if (nice > 0) ::setpriority(PRIO_PROCESS, static_cast<id_t>(::syscall(SYS_gettid)), nice);
        cudaSetDevice(ordinal);
        ScratchLease scratch;
        for (;;) {
            const size_t i = next->fetch_add(1);
            if (i >= pieces->size()) return;
            const Piece& pc = (*pieces)[i];
            try {
                const StagedFile& f = *pc.f;
                uint64_t piece_crc = 0;
                if (f.placement == Placement::hash) {
                    Crc64 c;
                    const int fd = ::open((dir / f.rel).c_str(), O_RDONLY | O_CLOEXEC);
                    require(fd >= 0, Errc::archive_corruption, "cannot open " + (dir / f.rel).string());
                    for (uint64_t done = 0; done < pc.len;) {
                        const ssize_t n = ::pread(fd, scratch.get(), std::min<uint64_t>(kScratch, pc.len - done),
                                                  static_cast<off_t>(pc.off + done));
                        if (n <= 0) {
                            ::close(fd);
                            raise(Errc::archive_corruption, "short read on " + (dir / f.rel).string());
                        }
                        c.update(scratch.get(), static_cast<size_t>(n));
                        done += static_cast<uint64_t>(n);
                    }
                    ::close(fd);
                    piece_crc = c.value();
                } else {
                    unsigned char* h = (f.placement == Placement::device ? hbase : pbase) + f.offset + pc.off;
                    read_range(dir / f.rel, h, pc.off, pc.len);
                    if (f.placement == Placement::host) piece_crc = crc64(h, pc.len);
                }
                std::lock_guard lock(sh->mu);  // one submission order on the streams
                if (f.placement == Placement::device) {
                    const uint32_t b0 = f.first_block + static_cast<uint32_t>(pc.off / kCrcBlockBytes);
                    const uint32_t nblk = static_cast<uint32_t>((pc.len + kCrcBlockBytes - 1) / kCrcBlockBytes);
                    cuda_check(cudaMemcpyAsync(dbase + f.offset + pc.off, hbase + f.offset + pc.off, pc.len,
                                               cudaMemcpyHostToDevice, copy),
                               "cudaMemcpyAsync(archive H2D)");
                    cudaEvent_t landed;
                    cuda_check(cudaEventCreateWithFlags(&landed, cudaEventDisableTiming), "cudaEventCreate");
                    cuda_check(cudaEventRecord(landed, copy), "cudaEventRecord");
                    cuda_check(cudaStreamWaitEvent(side, landed, 0), "cudaStreamWaitEvent");
                    cudaEventDestroy(landed);
                    cuda_check(fdy_launch_crc64_blocks(dbase, d_blocks + b0, nblk, d_crc + b0, d_len + b0, side),
                               "CRC block launch");
                } else {
                    sh->piece_crc[pc.slot] = piece_crc;
                    sh->piece_len[pc.slot] = pc.len;
                }
                if (--sh->pieces_left[f.segment] == 0) complete(f);
                if (--sh->remaining == 0) sh->read_ms = ms_since(sh->t0);
            } catch (...) {
                std::lock_guard lock(sh->mu);
                if (!sh->error) sh->error = std::current_exception();
                next->store(pieces->size());
            }
            sh->cv.notify_all();
        }
    };
    const unsigned nl = static_cast<unsigned>(std::min<size_t>(std::max(1u, lanes), std::max<size_t>(1, pieces->size())));
    for (unsigned l = 0; l < nl; ++l) sh_->lanes.emplace_back(body);
    trace_point("  staging: lanes started", sh_->t0);
    if (t) t->h2d_bytes += device_bytes_;
}

StagedArchive::~StagedArchive() {
    join();
    if (sh_) {
        cudaSetDevice(dev_.ordinal());
        cudaStreamSynchronize(dev_.copy_stream());  // nothing may still read the staging buffers
        cudaStreamSynchronize(dev_.side_stream());
        for (auto& e : sh_->done)
            if (e) cudaEventDestroy(e);
    }
}

void StagedArchive::join() {
    if (!sh_) return;
    for (auto& l : sh_->lanes)
        if (l.joinable()) l.join();
    sh_->lanes.clear();
}

const StagedFile& StagedArchive::file(const std::string& rel) const {
    auto it = files_.find(rel);
    require(it != files_.end(), Errc::archive_corruption, "archive has no " + rel);
    return it->second;
}

void StagedArchive::wait_ready(const StagedFile& f) const {
    std::unique_lock lock(sh_->mu);
    sh_->cv.wait(lock, [&] { return sh_->error || sh_->ready[f.segment]; });
    if (sh_->error) std::rethrow_exception(sh_->error);
}

uint64_t StagedArchive::digest_of(const StagedFile& f) const {
    if (f.placement != Placement::device) return sh_->cpu_digest[f.segment];
    cuda_check(cudaEventSynchronize(sh_->done[f.dseg]), "cudaEventSynchronize(CRC)");
    return reinterpret_cast<const uint64_t*>(digests_.data())[f.dseg];
}

void StagedArchive::order_after(const std::string& rel, cudaStream_t stream) {
    const StagedFile& f = file(rel);
    require(f.placement == Placement::device, Errc::invalid_argument, rel + " is not staged in HBM");
    wait_ready(f);
    cuda_check(cudaStreamWaitEvent(stream, sh_->done[f.dseg], 0), "cudaStreamWaitEvent");
}

void StagedArchive::verify_file(const Manifest& manifest, const std::string& rel, StageTimings* t) {
    const auto t0 = Clock::now();
    const StagedFile& f = file(rel);
    wait_ready(f);
    const uint64_t got = digest_of(f);
    if (t) t->integrity_ms += ms_since(t0);
    if (got != manifest.file_digests.at(rel)) verify(manifest, t);  // reports in manifest order
    require(got == manifest.file_digests.at(rel), Errc::archive_corruption, "integrity check failed for " + rel);
}

uint64_t StagedArchive::digest(const std::string& rel) const {
    const StagedFile& f = file(rel);
    wait_ready(f);
    return digest_of(f);
}

void StagedArchive::finish(StageTimings* t) {
    join();
    if (sh_->error) std::rethrow_exception(sh_->error);
    if (t) t->read_ms = std::max(t->read_ms, sh_->read_ms);
}

void StagedArchive::verify(const Manifest& manifest, StageTimings* t) {
    const auto t0 = Clock::now();
    join();
    if (sh_->error) std::rethrow_exception(sh_->error);
    if (t) t->read_ms += sh_->read_ms;
    for (const auto& [rel, digest] : manifest.file_digests)
        require(digest_of(file(rel)) == digest, Errc::archive_corruption, "integrity check failed for " + rel);
    if (t) t->integrity_ms += ms_since(t0);
}

std::span<const uint8_t> StagedArchive::host(const std::string& rel) const {
    const StagedFile& f = file(rel);
    require(f.placement != Placement::hash, Errc::invalid_argument, rel + " was hashed, not kept in host memory");
    wait_ready(f);
    return {(f.placement == Placement::device ? host_.data() : pageable_.data()) + f.offset, f.length};
}

const unsigned char* StagedArchive::device(const std::string& rel) const {
    const StagedFile& f = file(rel);
    require(f.placement == Placement::device, Errc::invalid_argument, rel + " is not staged in HBM");
    return device_.data() + f.offset;
}

uint64_t StagedArchive::size(const std::string& rel) const { return file(rel).length; }

// ------------------------------------------------------------------ materialize

namespace {

// Launches the fused kernel over the store and queues the D2H of the result.
struct Launched {
    DeviceBuffer out;
    MaterializeTiming mt;
    Clock::time_point t1, t2;
    uint64_t bytes = 0;
};

void launch_from_store(Device& dev, const Manifest& manifest, DeviceStore& store, const MaterializeRequest& req,
                       void* host_out, uint64_t cap, Launched& L) {
    const fdt_header& H = store.header;
    check_store_sources(H, manifest);
    if (host_out)
        require(cap >= H.members_image_bytes, Errc::invalid_argument,
                "output buffer holds " + std::to_string(cap) + " bytes, the member images need " +
                    std::to_string(H.members_image_bytes));
    L.out = DeviceBuffer(dev, std::max<uint64_t>(H.members_image_bytes, 16));
    L.mt.gate = false;  // part of a pipeline: no stream hold for the events
    launch_materialize(dev, store, req, L.out.data(), &L.mt);
    L.t2 = Clock::now();
    if (host_out) {
        dev.make_current();
        cuda_check(cudaMemcpyAsync(host_out, L.out.data(), H.members_image_bytes, cudaMemcpyDeviceToHost,
                                   dev.stream()),
                   "cudaMemcpyAsync(member images D2H)");
    }
    L.bytes = H.members_image_bytes;
}

}  // namespace

static uint64_t materialize_archive_early(Device& dev, const fs::path& root, const Manifest& manifest,
                                          std::unique_ptr<StagedArchive> early,
                                          std::future<std::unique_ptr<StagedArchive>> rest_future, StageTimings& st,
                                          Clock::time_point t_all, const MaterializeRequest& req,
                                          void* host_out, uint64_t cap, ArchiveMaterializeTimings* t,
                                          MaterializedArchive* keep) {
    std::unique_ptr<StagedArchive> rest;
    auto others = [&]() -> StagedArchive& {
        if (!rest) rest = rest_future.get();  // rethrows a listing / staging error
        return *rest;
    };
    // reference verify_archive_integrity (pipeline.cpp:411-417): the first
    // failing (or missing) file in manifest order names the error
    auto verify_all = [&] {
        for (const auto& [rel, digest] : manifest.file_digests) {
            StagedArchive& s = early->has(rel) ? *early : others();
            require(s.has(rel), Errc::archive_corruption, "cannot open " + (root / rel).string());
            require(s.digest(rel) == digest, Errc::archive_corruption, "integrity check failed for " + rel);
        }
    };
    Launched L;
    std::span<const uint8_t> host;
    std::optional<StoreView> view;
    std::exception_ptr bad_store;
    try {
        // the store's tables are validated as soon as its host copy is complete,
        // while its last pieces are still DMAed and CRCed; a validation error is
        // reported only once the digest has matched (integrity errors come first)
        host = early->host("templates.fdt");
        try {
            view.emplace(host);
        } catch (const Error&) {
            bad_store = std::current_exception();
        }
        trace_point("store tables validated", t_all);
        const auto ts = Clock::now();
        if (early->digest("templates.fdt") != manifest.file_digests.at("templates.fdt")) verify_all();
        st.integrity_ms += ms_since(ts);
        trace_point("store verified", t_all);
    } catch (const Error&) {
        rethrow_in_step("archive integrity");
    }
    if (bad_store) std::rethrow_exception(bad_store);
    L.t1 = Clock::now();
    early->order_after("templates.fdt", dev.stream());
    DeviceStore store = adopt_store(dev, early->device("templates.fdt"), host.size(), view->header());
    launch_from_store(dev, manifest, store, req, host_out, cap, L);
    trace_point("kernel launched", t_all);
    try {
        const auto tv = Clock::now();
        early->finish(&st);  // the kernel and the D2H are queued: the lanes hash the rest meanwhile
        others().finish(&st);
        verify_all();  // every file, while the D2H runs
        st.integrity_ms += ms_since(tv);
        trace_point("all files verified", t_all);
    } catch (const Error&) {
        cudaStreamSynchronize(dev.stream());
        rethrow_in_step("archive integrity");
    }
    cuda_check(cudaStreamSynchronize(dev.stream()), "cudaStreamSynchronize");
    trace_point("member images on the host", t_all);
    if (keep) {
        keep->images = std::move(L.out);
        keep->store_host.assign(host.begin(), host.end());
    }
    if (t) {
        t->read_ms = st.read_ms;
        t->integrity_ms = st.integrity_ms;
        t->crc_kernel_ms = st.crc_kernel_ms;
        t->materialize_ms = std::chrono::duration<double, std::milli>(L.t2 - L.t1).count();
        t->kernel_ms = L.mt.kernel_ms;
        t->d2h_ms = ms_since(L.t2);
        t->h2d_bytes = st.h2d_bytes;
        t->d2h_bytes = host_out ? L.bytes : 0;
        t->member_bytes = L.bytes;
        t->graphs = store.header.n_members;
        t->nodes = store.header.total_nodes;
        t->total_ms = ms_since(t_all);
    }
    return L.bytes;
}

uint64_t materialize_archive(Device& dev, const fs::path& root, const MaterializeRequest& req, unsigned lanes,
                             void* host_out, uint64_t cap, ArchiveMaterializeTimings* t, MaterializedArchive* keep) {
    const auto t_all = Clock::now();
    require(req.world >= 1 && req.rank < req.world, Errc::invalid_argument,
            "rank " + std::to_string(req.rank) + " is outside world size " + std::to_string(req.world));
    ArchivePaths paths{root};
    StageTimings st;
    // The store and graphs.bin (the largest file, hashed only) start streaming
    // before the manifest is parsed: the store -> kernel -> D2H chain and the
    // host hashing both begin at t = 0. Their digests are checked once the
    // manifest is known, in manifest order with every other file.
    // The store (to HBM, then kernel, then D2H) and every other archive file
    // (hashed on the host) start streaming before the manifest is parsed; the
    // digests are checked once it is known, in manifest order.
    std::unique_ptr<StagedArchive> early;
    std::future<std::unique_ptr<StagedArchive>> rest;
    {
        std::error_code e1;
        if (fs::is_regular_file(paths.template_store(), e1)) {
            StagePlan p;
            p.device = {"templates.fdt"};
            try {
                early = std::make_unique<StagedArchive>(dev, root, std::vector<std::string>{"templates.fdt"},
                                                        std::max(1u, std::min(lanes, 4u)), &st, p);
                // the rest: every other regular file under the archive directory
                // (extra files are hashed for nothing; missing ones are reported
                // against the manifest), listed and staged on a helper thread
                // on every lane, at the lowest CPU priority: while the store's
                // pieces are in flight the host is oversubscribed and the store
                // (the critical path: store -> kernel -> D2H) must win the cores
                // (tools/_exp_e2e_lanes.sh: median 4.2-4.3 ms vs 4.6-4.75 ms with
                // lanes - 4 at normal priority, and no 5.5-6 ms outliers)
                const unsigned rest_lanes = std::max(1u, lanes);
                rest = std::async(std::launch::async, [&dev, root, rest_lanes] {
                    std::vector<std::string> files;
                    const std::string prefix = root.string() + "/";
                    std::error_code ec;
                    for (auto it = fs::recursive_directory_iterator(root, ec);
                         !ec && it != fs::recursive_directory_iterator(); it.increment(ec)) {
                        if (!it->is_regular_file(ec)) continue;
                        const std::string full = it->path().string();
                        std::string rel = full.compare(0, prefix.size(), prefix) == 0 ? full.substr(prefix.size()) : full;
                        if (rel != "manifest" && rel != "templates.fdt") files.push_back(std::move(rel));
                    }
                    StagePlan background;
                    background.lane_nice = 19;
                    return std::make_unique<StagedArchive>(dev, root, files, rest_lanes, nullptr, background);
                });
            } catch (const Error&) {
                early.reset();  // the regular path reports it in manifest order
            }
        }
    }
    trace_point("early staging started", t_all);
    require(fs::exists(paths.manifest()), Errc::archive_corruption, "no manifest under " + root.string());
    const auto mb = slurp(paths.manifest());
    const Manifest manifest = parse_manifest(std::string(mb.begin(), mb.end()));
    trace_point("manifest parsed", t_all);
    if (early && manifest.file_digests.count("templates.fdt"))
        return materialize_archive_early(dev, root, manifest, std::move(early), std::move(rest), st, t_all, req,
                                         host_out, cap, t, keep);
    if (rest.valid()) {
        try {
            rest.get();
        } catch (...) {
        }
    }
    early.reset();
    std::unique_ptr<StagedArchive> staged;
    // the store (or, for a reference-written archive, the files it is packed
    // from) streams in first and is verified on its own; materialization and
    // the D2H of the result then overlap the reads of the remaining files,
    // whose verification still gates the return
    const bool has_store = manifest.file_digests.count("templates.fdt") != 0;
    // the store goes to HBM; a reference-written archive keeps the two files
    // it is packed from in host memory; every other file is only hashed
    StagePlan plan;
    std::vector<std::string> first;
    if (has_store) {
        plan.device = {"templates.fdt"};
        first = plan.device;
    } else {  // graphs.bin to HBM for the GPU packer; patch.bin first, parsed while graphs.bin streams
        plan.device = {"graphs.bin"};
        plan.host_first = {"patch.bin"};
        first = {"graphs.bin", "patch.bin"};
        if (manifest.file_digests.count("comm_slots.bin")) first.push_back("comm_slots.bin");
        plan.keep_host = [](const std::string& rel) { return rel == "patch.bin" || rel == "comm_slots.bin"; };
    }
    std::future<PatchView> patch_view;
    try {
        // a reference-written archive streams 188 MB where the store is 18 MB; the
        // stream is host-memory bound (page cache -> pinned at ~36 GB/s on 16
        // lanes). Half the lanes used to be faster while the patch-table parse
        // needed its cores for 5-7 ms; with the parse done by ~3 ms every lane
        // streams (tools/experiments/plain_lanes.sh, 16-core host, median of 5:
        // 8 lanes 14.7 / 16.0 ms, 12 lanes 14.6 / 13.9, 16 lanes 14.0 / 13.8).
        // FOUNDRY_PLAIN_STAGE_LANES overrides it for such sweeps.
        unsigned stage_lanes = lanes;
        if (const char* env = std::getenv("FOUNDRY_PLAIN_STAGE_LANES"); env && !has_store)
            stage_lanes = std::max(1, std::atoi(env));
        staged = std::make_unique<StagedArchive>(dev, root, manifest, stage_lanes, &st, plan);
        trace_point("staging started", t_all);
        if (!has_store && staged->has("patch.bin")) {
            // parse errors surface when the packer consumes it, after integrity
            patch_view = std::async(std::launch::async, [&staged, t_all] {
                const auto bytes = staged->host("patch.bin");
                trace_point("patch.bin on the host", t_all);
                PatchView v = parse_patch_view(bytes);
                trace_point("patch table parsed", t_all);
                return v;
            });
        }
        if (!has_store && std::getenv("FOUNDRY_DEBUG")) {
            (void)staged->host("graphs.bin");
            trace_point("graphs.bin read", t_all);
        }
        for (const auto& rel : first) staged->verify_file(manifest, rel, &st);
        trace_point("store verified", t_all);
    } catch (const Error&) {
        rethrow_in_step("archive integrity");
    }
    const auto t1 = Clock::now();
    DevicePackResult gpu;              // reference-written archive: packed now, on the GPU
    DevicePackTimings pack_t;
    std::span<const uint8_t> packed;   // its host copy
    DeviceStore store;
    if (has_store) {
        const auto host = staged->host("templates.fdt");
        const StoreView view(host);
        staged->order_after("templates.fdt", dev.stream());
        store = adopt_store(dev, staged->device("templates.fdt"), host.size(), view.header());
    } else {
        try {
            staged->order_after("graphs.bin", dev.stream());
            // keep: the caller gets the whole store on the host (fdy_load_members)
            gpu = pack_template_store_device(dev, staged->host("graphs.bin"), staged->device("graphs.bin"),
                                             staged->host("patch.bin"), manifest,
                                             staged->has("comm_slots.bin") ? staged->host("comm_slots.bin")
                                                                           : std::span<const uint8_t>{},
                                             nullptr, &pack_t, /*full_host_copy=*/keep != nullptr,
                                             &manifest.file_digests.at("graphs.bin"),
                                             patch_view.valid() ? &patch_view : nullptr);
            if (std::getenv("FOUNDRY_DEBUG"))
                std::fprintf(stderr,
                             "[foundry] pack phases: patch wait %.3f, prep %.3f, pass1 %.3f (uploaded %.3f, CRC queued %.3f, "
                             "synced %.3f; device: entry->kernels %.3f (scratch %.3f), kernels %.3f, CRC %.3f, read-back %.3f), host1 %.3f, pass2 %.3f (rank ops %.3f), "
                             "host2 %.3f (tiles %.3f), pass3 %.3f, total %.3f ms\n",
                             pack_t.patch_parse_ms, pack_t.prep_ms, pack_t.pass1_ms, pack_t.pass1_upload_ms,
                             pack_t.pass1_launch_ms, pack_t.pass1_sync_ms, pack_t.pass1_gpu_pre_ms, pack_t.pass1_gpu_alloc_ms,
                             pack_t.pass1_gpu_ms,
                             pack_t.pass1_gpu_crc_ms, pack_t.pass1_gpu_tail_ms,
                             pack_t.host1_ms, pack_t.pass2_ms,
                             pack_t.rank_ops_ms, pack_t.host2_ms, pack_t.tiles_ms, pack_t.pass3_ms, pack_t.total_ms);
        } catch (const Error&) {
            rethrow_in_step("template construction");
        }
        packed = gpu.host();
        store = adopt_store(dev, gpu.blob.data(), packed.size(), StoreView(packed).header());
        store.blob = std::move(gpu.blob);
    }
    const fdt_header& H = store.header;
    check_store_sources(H, manifest);
    if (host_out)
        require(cap >= H.members_image_bytes, Errc::invalid_argument,
                "output buffer holds " + std::to_string(cap) + " bytes, the member images need " +
                    std::to_string(H.members_image_bytes));
    DeviceBuffer out(dev, std::max<uint64_t>(H.members_image_bytes, 16));
    MaterializeTiming mt;
    mt.gate = false;  // part of a pipeline: no stream hold for the events
    launch_materialize(dev, store, req, out.data(), &mt);
    const auto t2 = Clock::now();
    trace_point("kernel launched", t_all);
    if (host_out) {
        dev.make_current();
        cuda_check(cudaMemcpyAsync(host_out, out.data(), H.members_image_bytes, cudaMemcpyDeviceToHost,
                                   dev.stream()),
                   "cudaMemcpyAsync(member images D2H)");
    }
    try {
        staged->verify(manifest, &st);  // every file, while the D2H runs
        trace_point("all files verified", t_all);
    } catch (const Error&) {
        cudaStreamSynchronize(dev.stream());
        rethrow_in_step("archive integrity");
    }
    cuda_check(cudaStreamSynchronize(dev.stream()), "cudaStreamSynchronize");
    trace_point("member images on the host", t_all);
    if (keep) {
        keep->images = std::move(out);
        const auto host = has_store ? staged->host("templates.fdt") : std::span<const uint8_t>(packed);
        keep->store_host.assign(host.begin(), host.end());
    }
    if (t) {
        t->read_ms = st.read_ms;
        t->integrity_ms = st.integrity_ms;
        t->crc_kernel_ms = st.crc_kernel_ms;
        t->materialize_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
        t->kernel_ms = mt.kernel_ms;
        t->d2h_ms = ms_since(t2);
        t->h2d_bytes = st.h2d_bytes;
        t->d2h_bytes = host_out ? H.members_image_bytes : 0;
        t->member_bytes = H.members_image_bytes;
        t->graphs = H.n_members;
        t->nodes = H.total_nodes;
        t->total_ms = ms_since(t_all);
    }
    return H.members_image_bytes;
}

}  // namespace foundry
