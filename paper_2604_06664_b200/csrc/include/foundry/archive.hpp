// Archive side-files: manifest (JSON), catalog.bin (FNDC), patch.bin (FNDP),
// memlayout.bin and the simulated device-binary format FNDB.
//
// Layouts and field names follow the reference so a reference-written archive
// loads here unchanged (reference pipeline.hpp:17-48, pipeline.cpp:23-139;
// binary_catalog.hpp:17-40, binary_catalog.cpp:33-105; rank_forge.hpp:19-38,
// rank_forge.cpp:43-102; det_alloc.hpp:18-53, det_alloc.cpp:20-59;
// kernel_image.hpp:11-61, kernel_image.cpp:14-117; templater.hpp:15-38).
#pragma once

#include <array>
#include <cstdint>
#include <string_view>
#include <filesystem>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "foundry/graph_model.hpp"

namespace foundry {

// ------------------------------------------------------------ allocator
struct RegionConfig {
    uint64_t base = 0x700000000000ull;
    uint64_t capacity = 4ull << 30;
    uint64_t granularity = 64ull << 10;
    bool operator==(const RegionConfig&) const = default;
};

enum class AllocWindow : uint8_t { pre_capture = 0, capture_window = 1 };

struct AllocationRecord {
    uint64_t sequence = 0;
    uint64_t size = 0;
    uint64_t address = 0;
    uint64_t length = 0;
    AllocWindow window = AllocWindow::pre_capture;
    bool operator==(const AllocationRecord&) const = default;
};

struct MemoryEventLog {
    RegionConfig config;
    uint64_t starting_offset = 0;
    uint64_t final_offset = 0;
    std::vector<AllocationRecord> records;
    bool operator==(const MemoryEventLog&) const = default;
};

std::vector<uint8_t> serialize_event_log(const MemoryEventLog& log);
MemoryEventLog parse_event_log(std::span<const uint8_t> bytes);

// ------------------------------------------------------------ grouping
struct TemplateGroup {
    TopologyKey key;
    uint32_t representative = 0;
    std::vector<uint32_t> members;
    std::vector<GraphLocator> locators;
    bool operator==(const TemplateGroup&) const = default;
};

struct GroupingManifest {
    std::vector<TemplateGroup> groups;
    uint32_t total_graphs = 0;
    uint32_t template_count = 0;
    double update_served_fraction() const {
        return total_graphs ? double(total_graphs - template_count) / total_graphs : 0.0;
    }
    bool operator==(const GroupingManifest&) const = default;
};

// Groups graphs by topology key; representative = smallest label
// (reference templater.cpp:18-52).
GroupingManifest group_graphs(const std::vector<CapturedGraph>& graphs);
void attach_locators(GroupingManifest& m, const std::vector<GraphLocator>& locators);

// ------------------------------------------------------------ manifest
struct Manifest {
    static constexpr uint32_t kFormatVersion = 1;
    uint32_t format_version = kFormatVersion;
    uint8_t hash_algorithm = kContentHashAlgorithm;
    uint64_t workload_digest = 0;
    std::string workload_text;
    RegionConfig allocator;
    uint64_t final_offset = 0;
    uint64_t kv_cache_bytes = 0;
    uint64_t comm_world_placeholder = 1;
    uint64_t comm_real_hash = 0;
    GroupingManifest grouping;
    std::string memlayout_ref = "memlayout.bin";
    std::string catalog_ref = "catalog.bin";
    std::string patch_table_ref = "patch.bin";
    std::map<std::string, uint64_t> file_digests;
    bool operator==(const Manifest&) const = default;
};

std::string serialize_manifest(const Manifest& m);
Manifest parse_manifest(const std::string& text);
// tests: 1 = parse_manifest's fast reader took the text and agrees with the full
// JSON parser, 0 = it took it and disagrees, -1 = it deferred to the full parser
int manifest_fast_path_agrees(const std::string& text);

struct ArchivePaths {
    std::filesystem::path root;
    std::filesystem::path manifest() const { return root / "manifest"; }
    std::filesystem::path graphs() const { return root / "graphs.bin"; }
    std::filesystem::path memlayout() const { return root / "memlayout.bin"; }
    std::filesystem::path catalog() const { return root / "catalog.bin"; }
    std::filesystem::path patch_table() const { return root / "patch.bin"; }
    std::filesystem::path binaries() const { return root / "binaries"; }
    std::filesystem::path binary(uint64_t hash) const { return binaries() / (hex16(hash) + ".bin"); }
    // B200 additions (ignored by the reference loader):
    std::filesystem::path template_store() const { return root / "templates.fdt"; }
    std::filesystem::path cubin(uint64_t hash) const {
        return binaries() / (hex16(hash) + ".sm_100a.cubin");
    }
    std::filesystem::path comm_slots() const { return root / "comm_slots.bin"; }
};

// ------------------------------------------------------------ FNDB images
struct KernelEntry {
    std::string name;
    uint32_t arg_buffer_size = 0;
    std::vector<uint32_t> hidden_offsets;  // 8-byte device addresses the kernel dereferences
    FuncAttrs attrs;
    bool operator==(const KernelEntry&) const = default;
};

struct KernelImage {
    bool relocatable = false;
    bool requires_device_init = false;
    uint32_t link_tag = 0;
    std::vector<KernelEntry> entrypoints;
    std::vector<uint8_t> aux;
    bool operator==(const KernelImage&) const = default;
};

std::vector<uint8_t> encode_kernel_image(const KernelImage& image);
KernelImage parse_kernel_image(std::span<const uint8_t> payload);
std::vector<uint8_t> link_segments(const std::vector<std::vector<uint8_t>>& segments);

// ------------------------------------------------------------ catalog
enum class LoadVariant : uint8_t { data = 0, file = 1, with_options = 2 };

struct KernelBinaryRecord {
    uint64_t hash = 0;
    LoadVariant variant = LoadVariant::data;
    std::vector<uint8_t> load_options;
    bool needs_device_init = false;
    bool is_stub = false;
    bool is_comm_real = false;
    std::vector<std::string> entrypoints;
    std::vector<FuncAttrs> entrypoint_attrs;
    bool operator==(const KernelBinaryRecord&) const = default;
};

struct Catalog {
    std::map<uint64_t, KernelBinaryRecord> binaries;
    bool operator==(const Catalog&) const = default;
};

std::vector<uint8_t> serialize_catalog(const Catalog& c);
Catalog parse_catalog(std::span<const uint8_t> bytes);

// ------------------------------------------------------------ patch table
struct CommPatchEntry {
    uint32_t node_id = 0;
    KernelRef stub;
    std::string real_name;
    std::vector<uint32_t> rank_offsets;
    std::vector<uint32_t> world_offsets;
    uint8_t patch_width = 8;
    bool operator==(const CommPatchEntry&) const = default;
};

struct PatchTable {
    uint64_t world_placeholder = 1;
    std::map<uint32_t, std::vector<CommPatchEntry>> per_graph;
    bool empty() const { return per_graph.empty(); }
    size_t total_entries() const;
    bool operator==(const PatchTable&) const = default;
};

std::vector<uint8_t> serialize_patch_table(const PatchTable& t);

// Zero-copy view of a patch table (same validation, same errors as
// parse_patch_table): entries point into the bytes, which must outlive it.
// LOAD reads the table through this (no per-entry allocations).
struct PatchEntryView {
    uint32_t node_id = 0;
    uint64_t stub_hash = 0;
    std::string_view stub_name, real_name;
    const uint8_t* rank_offsets = nullptr;  // n_rank little-endian u32
    const uint8_t* world_offsets = nullptr;
    uint32_t n_rank = 0, n_world = 0;
    uint8_t patch_width = 8;
    uint32_t rank_offset(uint32_t i) const;
    uint32_t world_offset(uint32_t i) const;
};
struct PatchView {
    uint64_t world_placeholder = 1;
    std::vector<PatchEntryView> entries;  // small tables (and the reference-order parse)
    // large tables: the entries live in a pooled block (a fresh 11 MB array costs
    // more in page faults than the parse; tools/experiments/patch_parse.py)
    std::shared_ptr<PatchEntryView> pooled;
    const PatchEntryView* entry_data() const { return pooled ? pooled.get() : entries.data(); }
    // label -> [first, first + count) in entries, sorted by label; the first
    // occurrence of a label wins (parse_patch_table's map emplace)
    std::vector<std::array<uint32_t, 3>> graphs;
    bool empty() const { return graphs.empty(); }
    std::span<const PatchEntryView> find(uint32_t label) const;  // empty span: none
    bool has(uint32_t label) const;
};
PatchView parse_patch_view(std::span<const uint8_t> bytes);
PatchTable parse_patch_table(std::span<const uint8_t> bytes);

// ------------------------------------------------------------ comm slots
// Per-rank communication state beyond rank/world (B200 addition, "comm_slots.bin",
// listed in the manifest digests so the reference loader only CRCs it). The
// stub layer authors the argument layout of every comm stub
// (rank_forge.cpp:18-22: rank@0 world@8 buf@16 payload@24) and so knows which
// bytes hold deployment state; a slot says "after apply_rank_patches, bytes
// [offset, offset + width) of node node_id's argument buffer := the low
// `width` bytes (little endian) of value table entry value_index". The value
// table (comm handles, peer buffer addresses, ...) is per rank and supplied at
// LOAD (LoadOptions::comm_values). Slots may only target nodes the patch table
// lists for the same graph (opaque compute kernels are never patched), are
// applied in table order after the rank/world writes, and may straddle
// 16-byte chunks. Format (little endian):
//   "FNDS" u16 version=1 u32 n_values u32 n_graphs
//   per graph: u32 label u32 count, per slot: u32 node_id u32 offset u32 value_index u8 width
struct CommSlot {
    uint32_t node_id = 0;
    uint32_t offset = 0;
    uint32_t value_index = 0;
    uint8_t width = 8;  // 1..8
    bool operator==(const CommSlot&) const = default;
};

struct CommSlotTable {
    uint32_t n_values = 0;  // value-table entries every rank must supply
    std::map<uint32_t, std::vector<CommSlot>> per_graph;  // keyed by batch label
    bool empty() const { return per_graph.empty(); }
    bool operator==(const CommSlotTable&) const = default;
};

std::vector<uint8_t> serialize_comm_slots(const CommSlotTable& t);
CommSlotTable parse_comm_slots(std::span<const uint8_t> bytes);

// The slot writes of one graph (host statement of the K3 value ops; the
// checks the packer performs): graph must already be rank-patched.
void apply_comm_slots(CapturedGraph& graph, std::span<const CommSlot> slots,
                      std::span<const CommPatchEntry> patches, std::span<const uint64_t> values);

// Host reference of the K3 rewrite (reference rank_forge.cpp:132-152), kept for
// the drop-in C++ surface; LOAD itself patches on the GPU.
void apply_rank_patches(CapturedGraph& graph, std::span<const CommPatchEntry> entries,
                        uint64_t real_comm_hash, uint32_t rank, uint32_t world);

}  // namespace foundry
