// Archive staging + GPU integrity + fused materialization: the data path the
// reference runs on CPU before any driver call — verify_archive_integrity
// (pipeline.cpp:411-417) and the PrepareFn over every member
// (pipeline.cpp:506-514) — as one host->HBM->host pipeline.
//
//   read   every manifest-listed file, `lanes` host threads, 8 MiB pieces,
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

struct StagedFile {
    std::string rel;
    uint64_t offset = 0;  // in host staging and in device staging
    uint64_t length = 0;
    uint32_t segment = 0;      // index in staging order
    uint32_t first_block = 0;  // CRC block table range
    uint32_t n_blocks = 0;
};

struct StageTimings {
    double read_ms = 0, integrity_ms = 0;  // integrity: wait for DMA + CRC kernel + compare
    float crc_kernel_ms = 0;
    uint64_t h2d_bytes = 0;
};

// All manifest-listed files, resident both in pinned host memory and in HBM,
// with their GPU CRC-64/XZ computed while they stream in:
//
//   reader lanes (host threads) take 8 MiB pieces in order — `first` files'
//   pieces before the rest — pread each into leased pinned staging, then on
//   the copy stream queue its H2D copy and the CRC of its 64 KiB blocks
//   (fdy_launch_crc64_blocks). The lane that submits a file's last piece
//   queues that file's fold and digest D2H (a `first` file) — the other
//   files fold in one batch after the last piece of all — and records the
//   file's event. So CRC overlaps the reads and the DMA; what is left when
//   the reads end is the last piece's copy + CRC and the folds.
//
// The constructor returns once the lanes are started; host(), device() and
// verify_*() wait for what they need.
class StagedArchive {
public:
    StagedArchive(Device& dev, const std::filesystem::path& root, const Manifest& manifest,
                  unsigned lanes, StageTimings* timings, std::vector<std::string> first = {});
    ~StagedArchive();
    StagedArchive(const StagedArchive&) = delete;
    StagedArchive& operator=(const StagedArchive&) = delete;

    // GPU CRC of every staged file against the manifest; raises
    // archive_corruption "integrity check failed for <rel>" on the first
    // mismatch in manifest order (caller adds the "archive integrity" step).
    void verify(const Manifest& manifest, StageTimings* timings);
    // The same for one file, without waiting for the others; on a mismatch
    // it reports the first failing file in manifest order, as verify() does.
    void verify_file(const Manifest& manifest, const std::string& rel, StageTimings* timings);
    // Makes `stream` wait until rel's bytes are in HBM and CRCed.
    void order_after(const std::string& rel, cudaStream_t stream);

    bool has(const std::string& rel) const { return files_.count(rel) != 0; }
    std::span<const uint8_t> host(const std::string& rel) const;  // waits for rel's reads
    const unsigned char* device(const std::string& rel) const;
    uint64_t size(const std::string& rel) const;
    uint64_t total_bytes() const { return total_; }

private:
    struct Shared;
    const StagedFile& file(const std::string& rel) const;
    void wait_submitted(const StagedFile& f) const;  // all of f's pieces queued (rethrows read errors)
    void join();

    Device& dev_;
    std::map<std::string, StagedFile> files_;
    std::vector<const StagedFile*> order_;  // staging order
    PinnedLease host_;
    DeviceBuffer device_;
    DeviceBuffer crc_;  // block table | block crc | block len | seg first | seg count | digests
    PinnedLease digests_;
    uint64_t total_ = 0;
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
uint64_t materialize_archive(Device& dev, const std::filesystem::path& root, uint32_t rank,
                             uint32_t world, uint64_t new_base, unsigned lanes, void* host_out,
                             uint64_t cap, ArchiveMaterializeTimings* timings);

}  // namespace foundry
