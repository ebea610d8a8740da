// Archive staging with overlapped reads + DMA, pinned pool, GPU integrity.
#include "foundry/staging.hpp"

#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <mutex>

#include <cuda_runtime.h>

#include "foundry/bytes.hpp"
#include "foundry/parallel.hpp"

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

StagedArchive::StagedArchive(Device& dev, const fs::path& root, const Manifest& manifest,
                             unsigned lanes, StageTimings* t)
    : dev_(dev) {
    const auto t0 = Clock::now();
    for (const auto& [rel, digest] : manifest.file_digests) {
        (void)digest;
        std::error_code ec;
        const uint64_t n = fs::file_size(root / rel, ec);
        require(!ec, Errc::archive_corruption, "cannot open " + (root / rel).string());
        files_[rel] = {rel, total_, n};
        total_ += (n + kAlign - 1) / kAlign * kAlign;
    }
    host_ = PinnedLease(dev, std::max<uint64_t>(total_, 16));
    device_ = DeviceBuffer(dev, std::max<uint64_t>(total_, 16));
    struct Piece {
        const StagedFile* f;
        uint64_t off, len;
    };
    std::vector<Piece> pieces;
    for (const auto& [rel, f] : files_)
        for (uint64_t o = 0; o < f.length; o += kPiece)
            pieces.push_back({&f, o, std::min<uint64_t>(kPiece, f.length - o)});
    // read a piece, then queue its DMA right away: reads and H2D overlap
    dev.make_current();
    cudaStream_t copy = dev.copy_stream();
    {  // device_ is stream-ordered on dev.stream(): the copies start after its allocation
        cudaEvent_t allocated;
        cuda_check(cudaEventCreateWithFlags(&allocated, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventRecord(allocated, dev.stream()), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(copy, allocated, 0), "cudaStreamWaitEvent");
        cudaEventDestroy(allocated);
    }
    parallel_for(pieces.size(), std::max(1u, lanes), [&](size_t i) {
        const Piece& pc = pieces[i];
        unsigned char* h = host_.data() + pc.f->offset + pc.off;
        read_range(root / pc.f->rel, h, pc.off, pc.len);
        cudaSetDevice(dev.ordinal());
        cuda_check(cudaMemcpyAsync(device_.data() + pc.f->offset + pc.off, h, pc.len,
                                   cudaMemcpyHostToDevice, copy),
                   "cudaMemcpyAsync(archive H2D)");
    });
    // the compute stream must see the staged bytes
    cudaEvent_t landed;
    cuda_check(cudaEventCreateWithFlags(&landed, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventRecord(landed, copy), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(dev.stream(), landed, 0), "cudaStreamWaitEvent");
    cudaEventDestroy(landed);
    if (t) {
        t->read_ms += ms_since(t0);
        t->h2d_bytes += total_;
    }
}

void StagedArchive::verify(const Manifest& manifest, StageTimings* t) {
    const auto t0 = Clock::now();
    std::vector<Segment> segs;
    std::vector<const std::string*> names;
    for (const auto& [rel, f] : files_) {
        segs.push_back({f.offset, f.length});
        names.push_back(&f.rel);
    }
    float ms = 0;
    const auto digests = crc64_device(dev_, device_.data(), segs, &ms);
    for (size_t i = 0; i < names.size(); ++i)
        require(digests[i] == manifest.file_digests.at(*names[i]), Errc::archive_corruption,
                "integrity check failed for " + *names[i]);
    if (t) {
        t->integrity_ms += ms_since(t0);
        t->crc_kernel_ms += ms;
    }
}

std::span<const uint8_t> StagedArchive::host(const std::string& rel) const {
    auto it = files_.find(rel);
    require(it != files_.end(), Errc::archive_corruption, "archive has no " + rel);
    return {host_.data() + it->second.offset, it->second.length};
}

const unsigned char* StagedArchive::device(const std::string& rel) const {
    auto it = files_.find(rel);
    require(it != files_.end(), Errc::archive_corruption, "archive has no " + rel);
    return device_.data() + it->second.offset;
}

uint64_t StagedArchive::size(const std::string& rel) const {
    auto it = files_.find(rel);
    require(it != files_.end(), Errc::archive_corruption, "archive has no " + rel);
    return it->second.length;
}

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
    try {
        staged = std::make_unique<StagedArchive>(dev, root, manifest, lanes, &st);
        staged->verify(manifest, &st);
    } catch (const Error&) {
        rethrow_in_step("archive integrity");
    }
    const auto t1 = Clock::now();
    std::vector<uint8_t> packed;  // reference-written archive: pack now
    DeviceStore store;
    if (staged->has("templates.fdt")) {
        const auto host = staged->host("templates.fdt");
        const StoreView view(host);
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
    DeviceBuffer out(dev, std::max<uint64_t>(H.members_image_bytes, 16));
    MaterializeRequest req;
    req.rank = rank;
    req.world = world;
    req.new_base = new_base;
    MaterializeTiming mt;
    launch_materialize(dev, store, req, out.data(), &mt);
    const auto t2 = Clock::now();
    if (host_out) {
        require(cap >= H.members_image_bytes, Errc::invalid_argument,
                "output buffer holds " + std::to_string(cap) + " bytes, the member images need " +
                    std::to_string(H.members_image_bytes));
        dev.make_current();
        cuda_check(cudaMemcpyAsync(host_out, out.data(), H.members_image_bytes, cudaMemcpyDeviceToHost,
                                   dev.stream()),
                   "cudaMemcpyAsync(member images D2H)");
        cuda_check(cudaStreamSynchronize(dev.stream()), "cudaStreamSynchronize");
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
