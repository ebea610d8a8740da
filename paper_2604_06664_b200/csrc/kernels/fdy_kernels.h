// Internal interface between the sm_100a kernels and the host runtime.
// (The public C-ABI is include/foundry_b200.h at the repository root.)
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "foundry/store_format.h"

struct FdyMaterializeArgs {
    const unsigned char* store;  // template store blob in HBM (never written)
    const unsigned char* tsrc;   // template source: tsrc + tile.src_off = the tile's
                                 // template chunks (store, or rtimg rebased by timage_base)
    unsigned char* out;          // member image arena in HBM
    unsigned char* rtimg;        // relocated-template scratch (timage_bytes), delta != 0
    const fdt_tile* tiles;
    const uint8_t* cmeta;
    const uint16_t* didx;
    const uint64_t* ddata;
    const fdt_rank_op* rops;
    const uint64_t* values;  // FDT_ROP_VALUE table (may be null)
    uint64_t timage_base;    // store offset of FDT_SEC_TIMAGES
    uint64_t timage_bytes;
    uint64_t old_base;       // captured VA base
    uint64_t span;           // final_offset
    uint64_t delta;          // new_base - old_base (mod 2^64)
    uint64_t rank;
    uint64_t world;
    uint32_t n_tiles;
    uint32_t n_values;
    uint32_t n_plain;  // tiles[0, n_plain) hold no relocatable template lane: read from the store
    uint32_t pad_;
};

// Device-side serve (kernels/serve.cu): one entry per template node.
struct FdyServeNode {
    void* devnode;          // cudaGraphDeviceNode_t of a device-updatable kernel node (else null)
    uint32_t param_bytes;   // the entry's argument-buffer size (what the node was built with)
    uint32_t kernel;        // store kernel index the node was built with
    uint32_t block[3];
    uint32_t shmem;
    int32_t memop_slot;     // memcpy / memset node: its index among the group's memops, else -1
    uint32_t pad;
};

// Serve plan, once per LOAD: for every member, whether the device can apply it
// (no node's function / block / shared memory differs from what its template
// was built with) and its memop records, so serve() needs no readback.
struct FdyServePlanArgs {
    const unsigned char* arena;              // member images in HBM
    const uint64_t* member_off;              // per member: image offset in the arena
    const uint32_t* member_group;            // per member: group index
    const FdyServeNode* const* group_nodes;  // per group: device serve table
    const uint32_t* group_n_nodes;
    const uint32_t* memop_base;              // per member: first slot in records
    uint8_t* member_host;                    // out, per member: 1 = host path needed
    uint64_t* records;                       // out: 3 x u64 per (member, memop slot)
    uint32_t n_members;
};

struct FdyServeArgs {
    const FdyServeNode* nodes;      // device table, n_nodes entries
    const unsigned char* image;     // member image in HBM (descriptors + pool)
    uint8_t* host_flags;            // host-mapped: 0 applied on device, 1 memop, 2 host path
    uint64_t* host_records;         // host-mapped: 3 x u64 per node (memop records)
    uint32_t* error_word;           // host-mapped: set to 1 when any device update fails, and
    uint8_t* member_failed;         //   member_failed[member] = 1 (per-member flags)
    uint32_t n_nodes;
    uint32_t member;
    uint32_t inject_failure;        // FaultInjection::fail_device_serve
};

// GPU packer (kernels/pack.cu): a reference-written archive's graphs.bin, in
// HBM, becomes the same FNDT template store the offline packer writes
// (host/template_store.cpp), decoded, diffed and compacted on the device.
// Members are numbered group-major in manifest order (the packer's order).
enum : uint32_t {
    FDY_PACK_DECODE = 1u,  // record fails to decode or validate: the host re-parses it for the message
    FDY_PACK_TOPO = 2u,    // topology differs from the group representative's
    FDY_PACK_PATCH = 4u,   // a patch entry / comm slot fails apply_rank_patches' checks
};

// A compacted kernel key as the host reads it back: binary hash u64 @0, func
// attrs 6 x i32 @8, name length u32 @32, name bytes @36 (only the first
// FDY_PACK_KEY_NAME bytes; longer names are read from the host copy).
#define FDY_PACK_KEY_BYTES 128u
#define FDY_PACK_KEY_NAME (FDY_PACK_KEY_BYTES - 36u)

struct FdyPackArgs {
    const unsigned char* graphs;  // graphs.bin in HBM
    uint64_t graphs_bytes;
    // per member
    const uint64_t* rec_off;      // record offset / length in graphs.bin (locator)
    const uint64_t* rec_len;
    const uint32_t* node_base;    // first global node index
    const uint32_t* n_nodes;      // node / edge counts from the record header (0 if unusable)
    const uint32_t* n_edges;
    const uint32_t* member_group;
    const uint64_t* out_off;      // pass 2: member image offset in the pack arena
    const uint32_t* tile_base;    // pass 2: first natural-order tile
    // per group
    const uint32_t* group_rep;    // member index of the representative
    const uint32_t* gnode_base;   // first per-(group, node) slot
    const uint64_t* g_image;      // pass 2: image bytes
    // per global node
    uint32_t* node_off;           // record-relative node offset (walk)
    uint32_t* node_member;        // member of the node (walk; ~0u = not decoded)
    uint32_t* node_slot;          // kernel-table slot (kernel nodes)
    // per (group, node)
    uint32_t* cap;                // max over the group of round16(blob length)
    const uint32_t* blob_off;     // pass 2: slot offset in the pool
    fdt_node_attrs* rep_attrs;    // the representative's launch attributes
    uint8_t* rep_type;            // the representative's node types
    // kernel table: open addressing over 64-bit key fingerprints
    unsigned long long* tkey;     // 0 = empty slot
    unsigned long long* tpos;     // min over the key's nodes of (member << 32 | node)
    uint32_t* tuniq;              // slot -> compacted index
    uint32_t tmask;
    uint32_t n_members;
    uint64_t seed;
    unsigned long long* upos;     // compacted: first position of each key
    uint64_t* uoff;               //            absolute graphs.bin offset of that node
    unsigned char* ukey;          //            its key bytes, FDY_PACK_KEY_BYTES each (see below)
    uint32_t* ucount;
    const uint32_t* ukidx;        // pass 2: compacted index -> store kernel index
    // patch entries (apply_rank_patches), flattened in member order
    const uint32_t* pe_node;      // global node of the stub (~0u: node id out of range)
    const uint64_t* pe_stub_hash;
    const uint32_t* pe_stub_name; // name ids into names / name_off / name_len
    const uint32_t* pe_real_name;
    const uint32_t* pe_need;      // argument bytes the entry's offsets and slots need
    uint32_t* pe_slot;            // kernel-table slot of the real comm kernel
    const uint32_t* entry_base;   // per member: first entry
    const unsigned char* names;
    const uint32_t* name_off;
    const uint32_t* name_len;
    uint64_t comm_real_hash;
    uint32_t n_entries;
    uint32_t total_nodes;
    uint32_t* status;             // per member: FDY_PACK_* bits
    uint32_t* flags;              // [0]: fingerprint collision
    // pass 2
    unsigned char* arena;         // member pack images (captured state + stub swaps)
    uint8_t* meta;                // FDT_CMETA_* per 16-byte chunk of arena
    const uint32_t* tile_member;  // per natural tile
    uint32_t* tile_count;         // diff entries per natural tile
    uint8_t* tile_reloc;          // 1: the tile's template chunks hold a relocatable lane
    const uint32_t* diff_lo;      // first diff entry per natural tile
    uint16_t* didx;               // store FDT_SEC_DIDX / FDT_SEC_DDATA
    uint64_t* ddata;
    uint32_t n_tiles;
    uint32_t pad_;
};

struct FdyCrcBlock {
    uint32_t segment;
    uint32_t length;   // <= kCrcBlockBytes
    uint64_t offset;   // absolute offset of the block in the device buffer
};

extern "C" {
size_t fdy_materialize_smem_bytes();
// A one-thread kernel that holds `stream` for `ns` ns (see materialize.cu).
cudaError_t fdy_launch_gate(cudaStream_t stream, uint64_t ns);
cudaError_t fdy_materialize_occupancy(int* blocks_per_sm);
// Measurement only: st.global.v4 fill of `bytes` at out (SMs x 8 CTAs).
cudaError_t fdy_launch_write_probe(unsigned char* out, uint64_t bytes, cudaStream_t stream);
// Measurement variant: relocation grid, then `between` recorded, then the member
// grid as an ordinary launch (events time the member pass alone).
cudaError_t fdy_launch_materialize_split(const FdyMaterializeArgs* args, int grid, cudaStream_t stream,
                                         cudaEvent_t between);
// delta == 0: one grid. Otherwise the template relocation grid, then the
// member grid under programmatic dependent launch (both on `stream`).
cudaError_t fdy_launch_materialize(const FdyMaterializeArgs* args, int grid, cudaStream_t stream);

// GPU packer passes (pack.cu), in stream order. Pass 1: walk (node offsets,
// record structure), fields (validation, topology, slot capacities, kernel
// keys), edges, verify (fingerprint collisions), compact (distinct keys).
// Pass 2 (after the host lays out groups and the kernel table): images, swaps,
// diff counts; pass 3: diff writes.
cudaError_t fdy_launch_pack_pass1(const FdyPackArgs* args, cudaStream_t stream);
cudaError_t fdy_launch_pack_pass2(const FdyPackArgs* args, cudaStream_t stream);
cudaError_t fdy_launch_pack_pass3(const FdyPackArgs* args, cudaStream_t stream);

// Chain fan-out (fanout.cu): publish `value` to a progress word (release,
// system scope) after everything before it on `stream`; hold `stream` until a
// (possibly peer-mapped) progress word reaches `value`.
// (not when *failed is set: a link that gave up stops forwarding; failed may be null)
cudaError_t fdy_launch_chain_publish(uint32_t* progress, uint32_t value, const uint32_t* failed,
                                     cudaStream_t stream);
// (gives up after timeout_ns, setting *failed)
cudaError_t fdy_launch_chain_wait(const uint32_t* progress, uint32_t value, uint64_t timeout_ns,
                                  uint32_t* failed, cudaStream_t stream);

// per device: x^(2^k) mod P and the constant-multiplier nibble tables built from them
cudaError_t fdy_crc64_set_constants(const uint64_t* x2k64);

// Device-side serve: apply a member image to a device-updatable exec (serve.cu).
// host_flags / host_records may be null (then nothing is written back).
cudaError_t fdy_launch_serve(const FdyServeArgs* args, cudaStream_t stream);
cudaError_t fdy_launch_serve_plan(const FdyServePlanArgs* args, cudaStream_t stream);
// CRC-64/XZ of n_segments byte ranges already resident in device memory.
// blocks: host-built table (see fdy_crc_plan) in device memory; partial /
// lengths scratch: n_blocks entries each; out: n_segments digests (device).
// The two halves of fdy_launch_crc64, for callers that CRC blocks as their
// bytes land (block i of the table -> block_crc[i], block_len[i]) and fold
// segments later. Block / segment pointers may be offset into larger tables.
cudaError_t fdy_launch_crc64_blocks(const unsigned char* base, const FdyCrcBlock* blocks,
                                    uint32_t n_blocks, uint64_t* block_crc, uint64_t* block_len,
                                    cudaStream_t stream);
cudaError_t fdy_launch_crc64_fold(const uint32_t* seg_first_block, const uint32_t* seg_n_blocks,
                                  uint32_t n_segments, uint64_t* block_crc, uint64_t* block_len,
                                  uint64_t* out, cudaStream_t stream);
cudaError_t fdy_launch_crc64(const unsigned char* base, const FdyCrcBlock* blocks,
                             uint32_t n_blocks, const uint32_t* seg_first_block,
                             const uint32_t* seg_n_blocks, uint32_t n_segments,
                             uint64_t* scratch_crc, uint64_t* scratch_len, uint64_t* out,
                             cudaStream_t stream);
}

inline constexpr uint32_t kCrcBlockBytes = 65536;  // one CTA, 8 KiB per warp
inline constexpr uint32_t kCrcMaxSegmentBlocks = (1u << 20) + 1;  // fold tables: 64 GiB per segment
