// Archive staging + GPU integrity + fused materialization: the data path the
// reference runs on CPU before any driver call — verify_archive_integrity
// (pipeline.cpp:411-417) and the PrepareFn over every member
// (pipeline.cpp:506-514) — as one host->HBM->host pipeline.
//
//   read   every manifest-listed file, `lanes` host threads, 2 MiB pieces,
//          into leased pinned staging; each piece is DMAed to HBM as soon as
//          it is read (reads and H2D overlap)
//   verify one GPU CRC-64/XZ launch over all files vs the manifest digests
//   expand the fused K2+K1+K3 kernel over the template store already in HBM
//
// Pinned staging comes from a per-process pool (a caching host allocator):
// the first materialization in a process pays cudaHostAlloc, later ones reuse.
#pragma once

#include <cstdint>
#include <filesystem>
#include <functional>
#include <map>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "foundry/archive.hpp"
#include "foundry/device.hpp"
#include "foundry/template_store.hpp"

namespace foundry {

// A pinned host buffer leased from the per-process pool; returns on destruction.
class PinnedLease {
public:
    PinnedLease() = default;
    PinnedLease(Device& dev, size_t bytes);
    ~PinnedLease();
    PinnedLease(PinnedLease&& o) noexcept { *this = std::move(o); }
    PinnedLease& operator=(PinnedLease&& o) noexcept;
    unsigned char* data() const { return p_; }
    size_t size() const { return n_; }

private:
    unsigned char* p_ = nullptr;
    size_t n_ = 0;
    size_t cap_ = 0;
    int device_ = -1;
};

// crc64_device split: launch() enqueues the plan upload, the kernel and the digests'
// read-back on dev.stream() and returns; digests() is valid once that stream has
// been synchronized past the launch (by the caller or by wait()).
// With `on` = another stream (dev.side_stream()), the work runs there, after
// everything already queued on dev.stream(); join(st) then makes `st` wait for it.
class CrcJob {
public:
    CrcJob() = default;
    ~CrcJob();
    CrcJob(const CrcJob&) = delete;
    CrcJob& operator=(const CrcJob&) = delete;
    void launch(Device& dev, const unsigned char* d_base, std::span<const Segment> segments,
                cudaStream_t on = nullptr);
    void join(cudaStream_t st);        // st waits for the launch (no-op on the launch stream)
    std::span<const uint64_t> wait();  // synchronizes the launch stream
    std::span<const uint64_t> digests() const { return {reinterpret_cast<const uint64_t*>(out_.data()), ns_}; }

private:
    Device* dev_ = nullptr;
    cudaStream_t on_ = nullptr;
    cudaEvent_t fork_ = nullptr, done_ = nullptr;
    DeviceBuffer scratch_;
    PinnedLease plan_, out_;
    size_t ns_ = 0;
};

// Pageable host memory leased from a per-process pool (the host-kept files'
// staging: no pinning cost, no page faults once warm); returns on destruction.
class PageableLease {
public:
    PageableLease() = default;
    explicit PageableLease(size_t bytes);
    ~PageableLease();
    PageableLease(PageableLease&& o) noexcept { *this = std::move(o); }
    PageableLease& operator=(PageableLease&& o) noexcept;
    unsigned char* data() const { return p_; }

private:
    unsigned char* p_ = nullptr;
    size_t cap_ = 0;
};

// Where a staged file goes. Every file is CRC-64/XZ-checked against the
// manifest; only the template store needs to be in HBM.
enum class Placement : uint8_t {
    device,  // pinned host copy + DMA to HBM; CRC on the GPU as its pieces land
    host,    // pageable host copy (the caller parses it); CRC on the host per piece
    hash,    // not kept: read through a per-lane scratch, CRC on the host
};

struct StagePlan {
    std::vector<std::string> device;                   // staged first, in this order
    std::function<bool(const std::string&)> keep_host;  // Placement::host files (others: hash)
    int lane_nice = 0;  // > 0: lanes run at this lower CPU priority (they yield to a concurrent
                        // critical-path stager when the host's cores are oversubscribed)
    std::vector<std::string> host_first;  // Placement::host files staged before the device files
                                          // (small inputs a consumer parses while the rest streams)
};

struct StagedFile {
    std::string rel;
    uint64_t offset = 0;  // device files: in pinned and device staging; host files: in pageable staging
    uint64_t length = 0;
    uint32_t segment = 0;  // index in staging order
    Placement placement = Placement::hash;
    uint32_t dseg = 0;         // device files: index of the GPU digest
    uint32_t first_block = 0;  // device files: CRC block table range
    uint32_t n_blocks = 0;
    uint32_t first_piece = 0;  // host / hash files: per-piece CRC slots
    uint32_t n_pieces = 0;
};

struct StageTimings {
    double read_ms = 0, integrity_ms = 0;  // integrity: waits for CRC results + compare
    float crc_kernel_ms = 0;
    uint64_t h2d_bytes = 0;
};

// All manifest-listed files, CRC-checked while they stream in:
//
//   reader lanes (host threads) take 2 MiB pieces in order — device files'
//   pieces first, then host-kept files, then hash-only ones. A device piece
//   is pread into leased pinned staging, then (in one submission order) its
//   H2D copy goes on the copy stream and the CRC of its 64 KiB blocks on the
//   side stream behind the copy (fdy_launch_crc64_blocks); the lane that
//   submits a device file's last piece queues its fold + digest D2H and
//   records the file's event. Host and hash pieces are CRCed on the lane
//   right after the read, while the bytes are still in cache (PCLMUL
//   folding, hash.hpp), and combined per file — bytes only the host needs
//   never cross PCIe.
//
// The constructor returns once the lanes are started; host(), device() and
// verify_*() wait for what they need.
class StagedArchive {
public:
    StagedArchive(Device& dev, const std::filesystem::path& root, const Manifest& manifest,
                  unsigned lanes, StageTimings* timings, StagePlan plan);
    // The same for an explicit file list (no manifest needed to start reading:
    // materialize_archive streams the store before the manifest is parsed).
    StagedArchive(Device& dev, const std::filesystem::path& root, const std::vector<std::string>& files,
                  unsigned lanes, StageTimings* timings, StagePlan plan);
    ~StagedArchive();
    StagedArchive(const StagedArchive&) = delete;
    StagedArchive& operator=(const StagedArchive&) = delete;

    // CRC of every staged file against the manifest; raises archive_corruption
    // "integrity check failed for <rel>" on the first mismatch in manifest
    // order (caller adds the "archive integrity" step).
    void verify(const Manifest& manifest, StageTimings* timings);
    // The same for one file, without waiting for the others; on a mismatch
    // it reports the first failing file in manifest order, as verify() does.
    void verify_file(const Manifest& manifest, const std::string& rel, StageTimings* timings);
    // Makes `stream` wait until a device file's bytes are in HBM and CRCed.
    void order_after(const std::string& rel, cudaStream_t stream);

    bool has(const std::string& rel) const { return files_.count(rel) != 0; }
    // CRC-64 of one staged file (waits for its pieces / GPU fold).
    uint64_t digest(const std::string& rel) const;
    // Joins the reader lanes (rethrows a read error); adds the read time.
    void finish(StageTimings* timings);
    // Host bytes of a device or host-kept file (waits for its reads).
    std::span<const uint8_t> host(const std::string& rel) const;
    const unsigned char* device(const std::string& rel) const;  // device files
    uint64_t size(const std::string& rel) const;
    uint64_t total_bytes() const { return total_; }

private:
    struct Shared;
    const StagedFile& file(const std::string& rel) const;
    void wait_ready(const StagedFile& f) const;  // all of f's pieces done (rethrows read errors)
    uint64_t digest_of(const StagedFile& f) const;
    void join();

    Device& dev_;
    std::map<std::string, StagedFile> files_;
    std::vector<const StagedFile*> order_;  // staging order
    PinnedLease host_;         // device files' pinned copies (the DMA source)
    PageableLease pageable_;   // host files (never DMAed: no pinning)
    DeviceBuffer device_;
    DeviceBuffer crc_;  // block table | block crc | block len | seg first | seg count | digests
    PinnedLease digests_;
    uint64_t total_ = 0;         // staged (device + host) bytes
    uint64_t device_bytes_ = 0;  // of which DMAed to HBM (pinned)
    uint64_t host_bytes_ = 0;    // of which host-kept (pageable)
    std::unique_ptr<Shared> sh_;
};

struct ArchiveMaterializeTimings {
    double total_ms = 0, read_ms = 0, integrity_ms = 0, materialize_ms = 0, d2h_ms = 0;
    float crc_kernel_ms = 0, kernel_ms = 0;
    uint64_t h2d_bytes = 0, d2h_bytes = 0, member_bytes = 0, graphs = 0, nodes = 0;
};

// The materialization path end to end: archive files -> pinned staging ->
// HBM -> GPU integrity -> fused K2+K1+K3 over every member for (rank, world,
// new_base) -> member images copied to host_out (if non-null; cap bytes).
// The GPU-native equivalent of the reference's verify_archive_integrity +
// PrepareFn over every member. Returns the member-image bytes.
// What a caller may keep of the materialization: the member images in HBM and
// a host copy of the store (its host sections decode the images).
struct MaterializedArchive {
    DeviceBuffer images;
    std::vector<uint8_t> store_host;
};

uint64_t materialize_archive(Device& dev, const std::filesystem::path& root, const MaterializeRequest& req,
                             unsigned lanes, void* host_out, uint64_t cap, ArchiveMaterializeTimings* timings,
                             MaterializedArchive* keep = nullptr);

}  // namespace foundry
