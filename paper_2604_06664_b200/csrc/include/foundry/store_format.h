/* store_format.h — the packed template store ("FNDT"), shared by the host
 * packer (csrc/host/template_store.cpp) and the sm_100a kernels
 * (csrc/kernels/materialize.cu). Plain C: no C++ or CUDA types.
 *
 * One store holds a whole archive's graph set as templates + diffs. It is
 * DMAed into HBM as a single blob and used in place; every offset below is a
 * byte offset from the start of the blob.
 *
 * Member image. Every member graph m of topology group g materializes into a
 * fixed-layout IMAGE of image_bytes(g) bytes (a multiple of 16):
 *
 *     [ node descriptors: n_nodes x fdt_node (48 B) ][ blob pool: pool_bytes ]
 *
 * Node n's argument bytes (kernel) or 24-byte memop record (memcpy:
 * src,dst,length / memset: dst,value,length) live at pool + node.blob_off,
 * blob_len bytes long; the slot capacity is the group-wide maximum rounded up
 * to 16 so every member of a group shares one layout. Bytes past blob_len are
 * zero. A template image is the group representative's image, unrelocated and
 * un-rank-patched (the captured state).
 *
 * Materialization of member m for (rank, world, new_base) =
 *   K2  copy the template image, replace the member's diff lanes;
 *   K1  for every 8-byte lane marked relocatable (template chunk meta, or the
 *       flag of the diff entry for a replaced lane) whose value v is in
 *       [old_base, old_base + final_offset): v += new_base - old_base;
 *   K3  apply the member's rank ops (rank / world u64 writes, per-rank
 *       value-table writes).
 * A diff entry exists for every 8-byte lane whose bytes OR relocation flag
 * differ from the template's, and carries the member's whole lane, so K1
 * commutes with K2: relocating the template images once per launch (3 MB)
 * and the diff lanes in registers gives the per-member result, and the
 * per-member pass is copy + scatter + rank ops.
 * The rank-independent part of apply_rank_patches (the stub -> real kernel
 * index swap) is applied at pack time, so it lives in the images; members of
 * a group whose rank ops for a tile are identical share one op range.
 * The kernel works tile by tile: a tile is up to tile_chunks consecutive
 * 16-byte chunks of one member image; the packer precomputes each tile's
 * diff and rank-op ranges so a CTA needs one descriptor load to start.
 * Tiles whose template chunks hold no relocatable lane are stored first
 * (n_plain_tiles of them): with delta != 0 they read the store directly
 * while the relocation grid is still running.
 * Comm slots (comm_slots.bin, archive.hpp) become FDT_ROP_VALUE ops after the
 * rank/world ops of the same chunk; the kernel reads values[aux] from the
 * caller's per-rank table of n_values entries.
 */
#ifndef FOUNDRY_STORE_FORMAT_H
#define FOUNDRY_STORE_FORMAT_H

#include <stdint.h>

#define FDT_VERSION 4u
#define FDT_TILE_CHUNKS 1024u /* 16 KiB of member image per tile */

enum fdt_section_id {
    FDT_SEC_GROUPS = 0,  /* fdt_group[n_groups]                         (host+device) */
    FDT_SEC_TIMAGES,     /* template images, 16-B aligned               (device)      */
    FDT_SEC_CMETA,       /* 1 byte per 16-B chunk of TIMAGES            (device)      */
    FDT_SEC_MEMBERS,     /* fdt_member[n_members]                       (host+device) */
    FDT_SEC_TILES,       /* fdt_tile[n_tiles]                           (device)      */
    FDT_SEC_DIDX,        /* u16 per diff entry: lane in tile | reloc    (device)      */
    FDT_SEC_DDATA,       /* u64 per diff entry: the member's lane value (device)      */
    FDT_SEC_ROPS,        /* fdt_rank_op[n_rank_ops]                     (device)      */
    FDT_SEC_KERNELS,     /* fdt_kernel[n_kernels]                       (host)        */
    FDT_SEC_NODEATTRS,   /* fdt_node_attrs per template node            (host)        */
    FDT_SEC_EDGES,       /* u32 pairs per group, concatenated           (host)        */
    FDT_SEC_STRINGS,     /* kernel names                                (host)        */
    FDT_NSEC
};

typedef struct {
    uint64_t offset;
    uint64_t bytes;
} fdt_section;

typedef struct {
    char magic[4]; /* "FNDT" */
    uint16_t version;
    uint16_t flags;
    uint32_t header_bytes;
    uint32_t n_groups;
    uint32_t n_members;
    uint32_t n_kernels;
    uint32_t n_tiles;
    uint32_t tile_chunks;
    uint32_t n_diffs;
    uint32_t n_rank_ops;
    uint64_t source_graphs_crc; /* graphs.bin digest this store was packed from */
    uint64_t source_patch_crc;  /* patch.bin digest */
    uint64_t old_base;          /* captured VA range: manifest allocator.base */
    uint64_t final_offset;      /*                    and final_offset        */
    uint64_t real_comm_hash;
    uint64_t members_image_bytes; /* sum of member image sizes = output arena */
    uint64_t total_nodes;         /* sum over members of node counts */
    /* v4 */
    uint32_t n_plain_tiles;    /* the first n_plain_tiles tiles read no relocatable
                                  template lane (they need not wait for K1's grid) */
    uint32_t n_values;         /* per-rank value-table entries FDT_ROP_VALUE ops read */
    uint64_t source_slots_crc; /* comm_slots.bin digest (0: no comm slots) */
    fdt_section sec[FDT_NSEC];
} fdt_header;

/* Node descriptor, 48 bytes, inside every image. */
typedef struct {
    uint8_t type; /* 0 kernel, 1 memcpy, 2 memset, 3 empty (graph_model.hpp NodeType) */
    uint8_t reserved0;
    uint16_t reserved1;
    uint32_t kernel; /* index into FDT_SEC_KERNELS (kernel nodes) */
    uint32_t grid[3];
    uint32_t block[3];
    uint32_t shmem;
    uint32_t blob_len;
    uint32_t blob_off; /* from the start of the pool */
    uint32_t reserved2;
} fdt_node;

typedef struct {
    uint64_t timage_off;  /* template image, from blob start */
    uint64_t image_bytes; /* per-member image size (desc + pool) */
    uint32_t n_nodes;
    uint32_t n_edges;
    uint32_t first_member; /* into FDT_SEC_MEMBERS */
    uint32_t n_members;
    uint32_t representative;
    uint32_t attrs_first; /* into FDT_SEC_NODEATTRS (n_nodes entries) */
    uint64_t edges_off;   /* byte offset within FDT_SEC_EDGES */
    uint64_t key_hi, key_lo; /* topology key (murmur3_x64_128) */
} fdt_group;

typedef struct {
    uint32_t label;
    uint32_t group;
    uint64_t out_off;  /* member image offset within the output arena */
    uint32_t first_tile;
    uint32_t n_tiles;
    uint32_t n_nodes;
    uint32_t pad;
} fdt_member;

typedef struct {
    uint64_t src_off;  /* template image chunk base, from blob start */
    uint64_t dst_off;  /* member image chunk base, from output arena start */
    uint32_t nchunks;  /* <= tile_chunks */
    uint32_t member;
    uint32_t diff_lo, diff_hi;   /* diff entries covering this tile */
    uint32_t rop_lo, rop_hi;     /* rank ops covering this tile */
    uint32_t chunk_base;         /* first chunk index (within the member image) */
    uint32_t pad;
} fdt_tile;

/* Diff entry index: the 8-byte lane's index within its tile (< 2 x
 * FDT_TILE_CHUNKS) and, in bit 15, the member lane's relocation flag. */
#define FDT_DIDX_LANE_MASK 0x7FFFu
#define FDT_DIDX_RELOC 0x8000u

#define FDT_CMETA_LANE0 0x1u /* bytes 0-7 of the chunk are a relocatable slot */
#define FDT_CMETA_LANE1 0x2u /* bytes 8-15 */

enum fdt_rank_op_kind {
    FDT_ROP_RANK = 0,   /* u64 rank   (CommPatchEntry.rank_offsets)  */
    FDT_ROP_WORLD = 1,  /* u64 world  (CommPatchEntry.world_offsets) */
    FDT_ROP_KERNEL = 2, /* u32 kernel index = aux (the packer folds the stub ->
                           real swap into the images instead; kept for stores
                           whose swap is rank-dependent) */
    FDT_ROP_VALUE = 3,  /* u64 per-rank value table[aux] (comm handles, peer buffers) */
};

/* One rank op touches bytes of ONE 16-byte chunk: for every set bit j of
 * mask, chunk byte j := byte (j - shift) of the little-endian value. An
 * unaligned u64 write spanning two chunks is two ops. */
typedef struct {
    uint32_t chunk; /* chunk index within the member image */
    uint8_t kind;
    int8_t shift;
    uint16_t mask;
    uint32_t aux;
    uint32_t pad;
} fdt_rank_op;

typedef struct {
    uint64_t binary_hash;
    uint32_t name_off; /* into FDT_SEC_STRINGS */
    uint32_t name_len;
    int32_t func_attrs[6];
} fdt_kernel;

typedef struct {
    uint32_t cluster[3];
    int32_t sched_policy;
    int32_t sync_default;
    int32_t sync_remote;
    uint32_t attr_query; /* bool */
} fdt_node_attrs;

#if FDT_TILE_CHUNKS * 2 > FDT_DIDX_LANE_MASK + 1
#error "tile lanes must fit the diff index"
#endif

#endif
