// Host side of the packed template store (format: foundry/store_format.h).
//
// pack_template_store() is the offline (SAVE-side) conversion of an archive's
// graphs.bin + patch.bin into templates + per-member diffs + rank ops. It runs
// the reference's own decode (parse_graph_at, graph_model.cpp:295-303) over
// every member and validates each patch entry exactly as apply_rank_patches
// would (rank_forge.cpp:132-152), so the store is parity-true by construction.
//
// StoreView is the LOAD-side, host-only view of a store blob: it parses the
// header and the host sections (kernel table, node attrs, edges) and can turn
// any materialized member image back into a CapturedGraph / FNDG record, which
// is how tests compare GPU output against the CPU oracle byte for byte.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "foundry/archive.hpp"
#include "foundry/graph_model.hpp"
#include "foundry/store_format.h"

namespace foundry {

struct PackStats {
    uint64_t template_bytes = 0;
    uint64_t diff_entries = 0;
    uint64_t rank_ops = 0;
    uint64_t member_image_bytes = 0;
    uint64_t store_bytes = 0;
};

// slots_bin: the archive's comm_slots.bin (empty: none).
std::vector<uint8_t> pack_template_store(std::span<const uint8_t> graphs_bin,
                                         std::span<const uint8_t> patch_bin,
                                         const Manifest& manifest, unsigned threads = 0,
                                         PackStats* stats = nullptr,
                                         std::span<const uint8_t> slots_bin = {});

// Packs an archive directory in place: writes templates.fdt and records its
// digest in the manifest (the archive stays loadable by the reference build,
// which only verifies the extra file's digest).
PackStats pack_archive_store(const std::filesystem::path& archive, unsigned threads = 0);

// The stub layer's authoring step for per-rank comm state (archive.hpp
// CommSlotTable): writes comm_slots.bin, records its digest in the manifest
// and re-packs templates.fdt when the archive has one. The table is validated
// against graphs.bin + patch.bin first (the packer's checks).
void write_comm_slots(const std::filesystem::path& archive, const CommSlotTable& table);

// The packer's rank-op emitter (shared with the GPU packer): a little-endian
// write of `width` bytes at image byte offset `at`, split into per-chunk ops.
namespace store_detail {
void emit_write(std::vector<fdt_rank_op>& ops, uint64_t at, uint32_t width, uint8_t kind, uint32_t aux);
}

class StoreView {
public:
    explicit StoreView(std::span<const uint8_t> blob);

    const fdt_header& header() const { return h_; }
    std::span<const uint8_t> blob() const { return blob_; }

    uint32_t n_groups() const { return h_.n_groups; }
    uint32_t n_members() const { return h_.n_members; }
    const fdt_group& group(uint32_t g) const { return groups_[g]; }
    const fdt_member& member(uint32_t m) const { return members_[m]; }
    const fdt_kernel& kernel(uint32_t k) const { return kernels_[k]; }
    std::string_view kernel_name(uint32_t k) const;
    KernelRef kernel_ref(uint32_t k) const;
    FuncAttrs kernel_func_attrs(uint32_t k) const;
    const fdt_node_attrs& node_attrs(uint32_t g, uint32_t n) const;
    std::span<const uint32_t> edges(uint32_t g) const;  // from,to pairs

    // Member index for a batch label, or -1.
    int64_t member_of(uint32_t label) const;

    // Node descriptors of a materialized member image stay inside the image
    // (type, kernel index, argument / memop bytes); archive-corruption otherwise.
    void check_image(uint32_t member, const uint8_t* image) const;

    // Decode a member image (the GPU's output layout) back to a graph.
    CapturedGraph image_to_graph(uint32_t member, std::span<const uint8_t> image) const;

private:
    void validate_tables() const;

    std::span<const uint8_t> blob_;
    fdt_header h_{};
    const fdt_group* groups_ = nullptr;
    const fdt_member* members_ = nullptr;
    const fdt_kernel* kernels_ = nullptr;
    const fdt_node_attrs* attrs_ = nullptr;
    const uint8_t* edges_ = nullptr;
    const char* strings_ = nullptr;
    std::vector<int32_t> by_label_;
    std::vector<std::pair<uint32_t, uint32_t>> sparse_labels_;  // (label, member) when labels are sparse
};

}  // namespace foundry
