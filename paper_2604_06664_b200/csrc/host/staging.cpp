// Archive staging with overlapped reads + DMA, pinned pool, GPU integrity.
#include "foundry/staging.hpp"

#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>

#include <cuda_runtime.h>

#include "foundry/bytes.hpp"
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
constexpr size_t kPiece = 8ull << 20;

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

// ------------------------------------------------------------------ staging

struct StagedArchive::Shared {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<uint32_t> pieces_left;       // per segment
    std::vector<cudaEvent_t> done;           // per segment, recorded after its fold
    std::vector<uint8_t> submitted;          // per segment
    std::exception_ptr error;                // first reader failure
    size_t remaining = 0;                    // pieces not yet submitted
    std::vector<std::thread> lanes;
    Clock::time_point t0;
    double read_ms = 0;
};

StagedArchive::StagedArchive(Device& dev, const fs::path& root, const Manifest& manifest,
                             unsigned lanes, StageTimings* t, std::vector<std::string> first)
    : dev_(dev), sh_(std::make_unique<Shared>()) {
    sh_->t0 = Clock::now();
    for (const auto& [rel, digest] : manifest.file_digests) {
        (void)digest;
        std::error_code ec;
        const uint64_t n = fs::file_size(root / rel, ec);
        require(!ec, Errc::archive_corruption, "cannot open " + (root / rel).string());
        files_[rel] = {rel, 0, n};
    }
    // staging order: the `first` files, then the rest in manifest order
    std::vector<uint8_t> is_first(files_.size(), 0);
    for (const auto& rel : first)
        if (files_.count(rel)) order_.push_back(&files_.at(rel));
    for (const auto& [rel, f] : files_)
        if (std::find(order_.begin(), order_.end(), &f) == order_.end()) order_.push_back(&f);
    const size_t n_first = std::min(first.size(), order_.size());
    std::vector<FdyCrcBlock> blocks;
    std::vector<uint32_t> seg_first, seg_count;
    for (size_t i = 0; i < order_.size(); ++i) {
        StagedFile& f = files_.at(order_[i]->rel);
        f.offset = total_;
        f.segment = static_cast<uint32_t>(i);
        f.first_block = static_cast<uint32_t>(blocks.size());
        for (uint64_t o = 0; o < f.length; o += kCrcBlockBytes)
            blocks.push_back({f.segment, static_cast<uint32_t>(std::min<uint64_t>(kCrcBlockBytes, f.length - o)),
                              f.offset + o});
        f.n_blocks = static_cast<uint32_t>(blocks.size()) - f.first_block;
        seg_first.push_back(f.first_block);
        seg_count.push_back(f.n_blocks);
        total_ += (f.length + kAlign - 1) / kAlign * kAlign;
    }
    const size_t nb = blocks.size(), ns = order_.size();
    host_ = PinnedLease(dev, std::max<uint64_t>(total_, 16));
    device_ = DeviceBuffer(dev, std::max<uint64_t>(total_, 16));
    // CRC scratch: block table | crc | len | first | count | digests
    const size_t table = nb * sizeof(FdyCrcBlock), plan = table + 2 * ns * 4;
    crc_ = DeviceBuffer(dev, plan + 2 * nb * 8 + ns * 8 + 64);
    digests_ = PinnedLease(dev, std::max<size_t>(plan, ns * 8) + 64);
    std::memcpy(digests_.data(), blocks.data(), table);
    std::memcpy(digests_.data() + table, seg_first.data(), ns * 4);
    std::memcpy(digests_.data() + table + ns * 4, seg_count.data(), ns * 4);
    auto* d_blocks = reinterpret_cast<FdyCrcBlock*>(crc_.data());
    auto* d_first = reinterpret_cast<uint32_t*>(crc_.data() + table);
    auto* d_count = d_first + ns;
    auto* d_crc = reinterpret_cast<uint64_t*>(crc_.data() + (plan + 7) / 8 * 8);
    auto* d_len = d_crc + nb;
    auto* d_out = d_len + nb;

    dev.make_current();
    cudaStream_t copy = dev.copy_stream();
    {  // device buffers are stream-ordered on dev.stream(): copies start after the allocations
        cudaEvent_t allocated;
        cuda_check(cudaEventCreateWithFlags(&allocated, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventRecord(allocated, dev.stream()), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(copy, allocated, 0), "cudaStreamWaitEvent");
        cudaEventDestroy(allocated);
    }
    cuda_check(cudaMemcpyAsync(crc_.data(), digests_.data(), plan, cudaMemcpyHostToDevice, copy),
               "cudaMemcpyAsync(CRC plan H2D)");
    // the plan must land before the digest slots (same pinned buffer) are reused
    cuda_check(cudaStreamSynchronize(copy), "cudaStreamSynchronize(CRC plan)");

    struct Piece {
        const StagedFile* f;
        uint64_t off, len;
    };
    auto pieces = std::make_shared<std::vector<Piece>>();
    for (const StagedFile* f : order_)
        for (uint64_t o = 0; o < f->length; o += kPiece)
            pieces->push_back({f, o, std::min<uint64_t>(kPiece, f->length - o)});
    sh_->pieces_left.assign(ns, 0);
    for (const Piece& pc : *pieces) ++sh_->pieces_left[pc.f->segment];
    sh_->submitted.assign(ns, 0);
    sh_->done.assign(ns, nullptr);
    for (auto& e : sh_->done) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    sh_->remaining = pieces->size();
    uint64_t* h_digest = reinterpret_cast<uint64_t*>(digests_.data());  // plan is no longer needed

    // folds one segment range and copies its digests to the pinned slots
    // CRC work runs on the side stream, each piece's blocks gated by an event
    // on its copy, so the copy engine streams pieces back to back
    cudaStream_t side = dev.side_stream();
    auto fold = [=](uint32_t s0, uint32_t n) {
        cuda_check(fdy_launch_crc64_fold(d_first + s0, d_count + s0, n, d_crc, d_len, d_out + s0, side),
                   "CRC fold launch");
        cuda_check(cudaMemcpyAsync(h_digest + s0, d_out + s0, 8ull * n, cudaMemcpyDeviceToHost, side),
                   "cudaMemcpyAsync(digest D2H)");
    };
    // empty files: fold + event right away (no pieces)
    for (uint32_t s = 0; s < ns; ++s)
        if (sh_->pieces_left[s] == 0 && s < n_first) {
            fold(s, 1);
            cuda_check(cudaEventRecord(sh_->done[s], side), "cudaEventRecord");
            sh_->submitted[s] = 1;
        }
    auto next = std::make_shared<std::atomic<size_t>>(0);
    Shared* sh = sh_.get();
    unsigned char* hbase = host_.data();
    unsigned char* dbase = device_.data();
    const int ordinal = dev.ordinal();
    const fs::path dir = root;  // the lanes outlive this constructor
    auto body = [=]() {
        cudaSetDevice(ordinal);
        for (;;) {
            const size_t i = next->fetch_add(1);
            if (i >= pieces->size()) return;
            const Piece& pc = (*pieces)[i];
            try {
                unsigned char* h = hbase + pc.f->offset + pc.off;
                read_range(dir / pc.f->rel, h, pc.off, pc.len);
                const uint32_t b0 = pc.f->first_block + static_cast<uint32_t>(pc.off / kCrcBlockBytes);
                const uint32_t nblk = static_cast<uint32_t>((pc.len + kCrcBlockBytes - 1) / kCrcBlockBytes);
                std::lock_guard lock(sh->mu);  // one submission order on the copy stream
                cuda_check(cudaMemcpyAsync(dbase + pc.f->offset + pc.off, h, pc.len, cudaMemcpyHostToDevice, copy),
                           "cudaMemcpyAsync(archive H2D)");
                cudaEvent_t landed;
                cuda_check(cudaEventCreateWithFlags(&landed, cudaEventDisableTiming), "cudaEventCreate");
                cuda_check(cudaEventRecord(landed, copy), "cudaEventRecord");
                cuda_check(cudaStreamWaitEvent(side, landed, 0), "cudaStreamWaitEvent");
                cudaEventDestroy(landed);
                cuda_check(fdy_launch_crc64_blocks(dbase, d_blocks + b0, nblk, d_crc + b0, d_len + b0, side),
                           "CRC block launch");
                const uint32_t s = pc.f->segment;
                if (--sh->pieces_left[s] == 0 && s < n_first) {
                    fold(s, 1);
                    cuda_check(cudaEventRecord(sh->done[s], side), "cudaEventRecord");
                    sh->submitted[s] = 1;
                }
                if (--sh->remaining == 0) {  // the rest fold in one launch
                    if (ns > n_first) fold(static_cast<uint32_t>(n_first), static_cast<uint32_t>(ns - n_first));
                    for (size_t k = n_first; k < ns; ++k) {
                        cuda_check(cudaEventRecord(sh->done[k], side), "cudaEventRecord");
                        sh->submitted[k] = 1;
                    }
                    sh->read_ms = ms_since(sh->t0);
                }
            } catch (...) {
                std::lock_guard lock(sh->mu);
                if (!sh->error) sh->error = std::current_exception();
                next->store(pieces->size());
            }
            sh->cv.notify_all();
        }
    };
    if (pieces->empty()) {
        for (size_t k = n_first; k < ns; ++k) {
            fold(static_cast<uint32_t>(k), 1);
            cuda_check(cudaEventRecord(sh_->done[k], side), "cudaEventRecord");
            sh_->submitted[k] = 1;
        }
    }
    const unsigned nl = static_cast<unsigned>(std::min<size_t>(std::max(1u, lanes), std::max<size_t>(1, pieces->size())));
    for (unsigned l = 0; l < nl; ++l) sh_->lanes.emplace_back(body);
    if (t) t->h2d_bytes += total_;
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

void StagedArchive::wait_submitted(const StagedFile& f) const {
    std::unique_lock lock(sh_->mu);
    sh_->cv.wait(lock, [&] { return sh_->error || sh_->submitted[f.segment]; });
    if (sh_->error) std::rethrow_exception(sh_->error);
}

void StagedArchive::order_after(const std::string& rel, cudaStream_t stream) {
    const StagedFile& f = file(rel);
    wait_submitted(f);
    cuda_check(cudaStreamWaitEvent(stream, sh_->done[f.segment], 0), "cudaStreamWaitEvent");
}

void StagedArchive::verify_file(const Manifest& manifest, const std::string& rel, StageTimings* t) {
    const auto t0 = Clock::now();
    const StagedFile& f = file(rel);
    wait_submitted(f);
    cuda_check(cudaEventSynchronize(sh_->done[f.segment]), "cudaEventSynchronize(CRC)");
    const uint64_t got = reinterpret_cast<const uint64_t*>(digests_.data())[f.segment];
    if (t) t->integrity_ms += ms_since(t0);
    if (got != manifest.file_digests.at(rel)) verify(manifest, t);  // reports in manifest order
    require(got == manifest.file_digests.at(rel), Errc::archive_corruption, "integrity check failed for " + rel);
}

void StagedArchive::verify(const Manifest& manifest, StageTimings* t) {
    const auto t0 = Clock::now();
    join();
    if (sh_->error) std::rethrow_exception(sh_->error);
    if (t) t->read_ms += sh_->read_ms;
    cuda_check(cudaStreamSynchronize(dev_.side_stream()), "cudaStreamSynchronize(CRC)");
    const auto* got = reinterpret_cast<const uint64_t*>(digests_.data());
    for (const auto& [rel, digest] : manifest.file_digests)
        require(got[file(rel).segment] == digest, Errc::archive_corruption, "integrity check failed for " + rel);
    if (t) t->integrity_ms += ms_since(t0);
}

std::span<const uint8_t> StagedArchive::host(const std::string& rel) const {
    const StagedFile& f = file(rel);
    wait_submitted(f);
    return {host_.data() + f.offset, f.length};
}

const unsigned char* StagedArchive::device(const std::string& rel) const {
    return device_.data() + file(rel).offset;
}

uint64_t StagedArchive::size(const std::string& rel) const { return file(rel).length; }

// ------------------------------------------------------------------ materialize

uint64_t materialize_archive(Device& dev, const fs::path& root, uint32_t rank, uint32_t world,
                             uint64_t new_base, unsigned lanes, void* host_out, uint64_t cap,
                             ArchiveMaterializeTimings* t) {
    const auto t_all = Clock::now();
    require(world >= 1 && rank < world, Errc::invalid_argument,
            "rank " + std::to_string(rank) + " is outside world size " + std::to_string(world));
    ArchivePaths paths{root};
    require(fs::exists(paths.manifest()), Errc::archive_corruption, "no manifest under " + root.string());
    const auto mb = slurp(paths.manifest());
    const Manifest manifest = parse_manifest(std::string(mb.begin(), mb.end()));
    StageTimings st;
    std::unique_ptr<StagedArchive> staged;
    // the store (or, for a reference-written archive, the files it is packed
    // from) streams in first and is verified on its own; materialization and
    // the D2H of the result then overlap the reads of the remaining files,
    // whose verification still gates the return
    const bool has_store = manifest.file_digests.count("templates.fdt") != 0;
    const std::vector<std::string> first =
        has_store ? std::vector<std::string>{"templates.fdt"} : std::vector<std::string>{"graphs.bin", "patch.bin"};
    try {
        staged = std::make_unique<StagedArchive>(dev, root, manifest, lanes, &st, first);
        for (const auto& rel : first) staged->verify_file(manifest, rel, &st);
    } catch (const Error&) {
        rethrow_in_step("archive integrity");
    }
    const auto t1 = Clock::now();
    std::vector<uint8_t> packed;  // reference-written archive: pack now
    DeviceStore store;
    if (has_store) {
        const auto host = staged->host("templates.fdt");
        const StoreView view(host);
        staged->order_after("templates.fdt", dev.stream());
        store = adopt_store(dev, staged->device("templates.fdt"), host.size(), view.header());
    } else {
        try {
            packed = pack_template_store(staged->host("graphs.bin"), staged->host("patch.bin"), manifest,
                                         lanes);
        } catch (const Error&) {
            rethrow_in_step("template construction");
        }
        store = upload_store(dev, packed.data(), packed.size());
        st.h2d_bytes += packed.size();
    }
    const fdt_header& H = store.header;
    require(H.source_graphs_crc == manifest.file_digests.at("graphs.bin") &&
                H.source_patch_crc == manifest.file_digests.at("patch.bin"),
            Errc::archive_corruption, "template store was packed from a different graphs.bin/patch.bin");
    if (H.n_rank_ops > 0)
        require(manifest.comm_real_hash != 0, Errc::unresolved_kernel,
                "archive carries comm patches but no real comm binary");
    if (host_out)
        require(cap >= H.members_image_bytes, Errc::invalid_argument,
                "output buffer holds " + std::to_string(cap) + " bytes, the member images need " +
                    std::to_string(H.members_image_bytes));
    DeviceBuffer out(dev, std::max<uint64_t>(H.members_image_bytes, 16));
    MaterializeRequest req;
    req.rank = rank;
    req.world = world;
    req.new_base = new_base;
    MaterializeTiming mt;
    mt.gate = false;  // part of a pipeline: no stream hold for the events
    launch_materialize(dev, store, req, out.data(), &mt);
    const auto t2 = Clock::now();
    if (host_out) {
        dev.make_current();
        cuda_check(cudaMemcpyAsync(host_out, out.data(), H.members_image_bytes, cudaMemcpyDeviceToHost,
                                   dev.stream()),
                   "cudaMemcpyAsync(member images D2H)");
    }
    try {
        staged->verify(manifest, &st);  // every file, while the D2H runs
    } catch (const Error&) {
        cudaStreamSynchronize(dev.stream());
        rethrow_in_step("archive integrity");
    }
    cuda_check(cudaStreamSynchronize(dev.stream()), "cudaStreamSynchronize");
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
