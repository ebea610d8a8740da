// GPU packer (kernels/pack.cu + host/device_pack.cpp): the FNDT template
// store that pack_template_store (template_store.hpp) writes offline, built on
// the device from an archive's graphs.bin already resident in HBM, for
// archives written by the reference (no templates.fdt).
#pragma once

#include <cstdint>
#include <future>
#include <memory>
#include <span>
#include <vector>

#include "foundry/archive.hpp"
#include "foundry/device.hpp"
#include "foundry/template_store.hpp"

namespace foundry {

struct DevicePackTimings {
    double prep_ms = 0;   // patch table view, member / group / entry tables
    double patch_parse_ms = 0;  // of which: the patch table view
    double pass1_ms = 0;  // upload + walk/fields/edges/verify/compact + record CRCs
    double pass1_upload_ms = 0, pass1_launch_ms = 0, pass1_sync_ms = 0;  // stamps within pass 1
    double pass1_gpu_ms = 0, pass1_gpu_crc_ms = 0;  // device time of pass 1 / its CRCs (FOUNDRY_DEBUG)
    double pass1_gpu_pre_ms = 0, pass1_gpu_tail_ms = 0, pass1_gpu_alloc_ms = 0;  // device: pass-1 entry -> kernels; kernels -> read-back done
    double host1_ms = 0;  // checks, kernel table, layout, rank ops
    double checks_ms = 0, kernel_table_ms = 0, rank_ops_ms = 0;  // of which
    double pass2_ms = 0;  // images + diff counts
    double host2_ms = 0;  // tile table, host sections
    double tiles_ms = 0;  // of which: the tile table and shared rank-op ranges
    double layout_ms = 0; //           header and section layout
    double pass3_ms = 0;  // diff writes + template images + D2H of the device sections
    double total_ms = 0;
    uint32_t kernel_keys = 0;  // distinct kernel keys the GPU table found
    uint32_t retries = 0;      // fingerprint collisions resolved by a reseed
};

struct DevicePackResult {
    // The store on the host, byte-identical to pack_template_store's when
    // host_complete; otherwise the device-only sections (template images, chunk
    // meta, diff streams: what only the kernels read) are not copied back and
    // their host bytes are unspecified. Host-side readers (StoreView) only use
    // the header and the host sections.
    std::unique_ptr<uint8_t[]> host_bytes;
    size_t host_size = 0;
    bool host_complete = false;
    DeviceBuffer blob;  // the whole store in HBM
    std::span<const uint8_t> host() const { return {host_bytes.get(), host_size}; }
};

// patch_view: patch_bin already being parsed (parse_patch_view) on another
// thread while graphs.bin streamed in; its errors surface here.
// verified_graphs_crc: graphs.bin's digest when the caller has already checked
// it and the other inputs against the manifest (LOAD's integrity pass); the
// header then takes the manifest digests; otherwise they are computed.
// graphs_host / d_graphs: graphs.bin on the host and in HBM (the device copy
// is read by the kernels; the host copy only for per-group and per-kernel
// metadata and, on error paths, to re-derive the reference's exact message for
// the failing record). Asynchronous work runs on dev.stream(); returns after a
// synchronize.
DevicePackResult pack_template_store_device(Device& dev, std::span<const uint8_t> graphs_host,
                                            const unsigned char* d_graphs, std::span<const uint8_t> patch_bin,
                                            const Manifest& manifest, std::span<const uint8_t> slots_bin = {},
                                            PackStats* stats = nullptr, DevicePackTimings* timings = nullptr,
                                            bool full_host_copy = true,
                                            const uint64_t* verified_graphs_crc = nullptr,
                                            std::future<PatchView>* patch_view = nullptr);

// The same for an archive directory: reads and uploads graphs.bin, packs it on
// the GPU, returns the store bytes (the tests compare them with the offline
// packer's; LOAD and fdy_prepare_archive use the staged path above).
std::vector<uint8_t> pack_archive_store_device(Device& dev, const std::filesystem::path& archive,
                                               DevicePackTimings* timings = nullptr);

}  // namespace foundry
