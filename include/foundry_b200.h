/* foundry_b200.h — C-ABI of the B200-native Foundry LOAD path.
 *
 * Plain C: opaque handles, pointers and sizes; no C++ or torch types. This is
 * the drop-in boundary a foreign binding (ctypes / cgo / JNI / N-API) binds,
 * exported by paper_2604_06664_b200/libfoundry_b200.so. INTEGRATION.md shows
 * the reference-side bindings.
 *
 * Two layers:
 *
 *  1. Session API — the reference's public LOAD surface, one call per
 *     reference entry point (reference proj/bindings/module.cpp:53-60,102-134
 *     and proj/include/foundry/pipeline.hpp:80-119):
 *       fdy_load                 <- foundry::load(archive, LoadOptions)      pipeline.hpp:116-119
 *       fdy_serving_replay       <- ServingContext::replay(batch)            pipeline.hpp:94
 *                                   + LaunchTrace::to_text                   sim_driver.cpp:21-38
 *       fdy_serving_batches      <- ServingContext::batches()                pipeline.hpp:95
 *       fdy_serving_counter(s)   <- ServingContext::counters()               pipeline.hpp:100
 *       fdy_serving_template_count <- ServingHandle.template_count           module.cpp:32
 *       fdy_serving_close        <- ~ServingContext
 *       fdy_serving_save_captured   GPU-side SAVE of a whole archive (reference save,
 *                                   pipeline.cpp:249-405) from device captures
 *       fdy_serving_capture_graph   GPU-side SAVE: the batch's graph
 *                                   stream-captured on the device and extracted back,
 *                                   as the FNDG record encode_graph_record writes
 *                                   (reference graph_model.cpp:205-218; capture
 *                                   semantics sim_driver.cpp:222-290)
 *
 *  2. Kernel API — the per-member work of the reference PrepareFn
 *     (pipeline.cpp:506-514: parse_graph_at graph_model.cpp:295-303 +
 *     apply_rank_patches rank_forge.cpp:132-152) and the archive integrity
 *     pass (verify_archive_integrity pipeline.cpp:411-417), moved onto the GPU:
 *       fdy_device_open / fdy_device_close
 *       fdy_store_upload      pinned/pageable host -> HBM DMA of a template store
 *       fdy_store_fanout      GPU -> GPU copy of a resident store (NVLink P2P)
 *       fdy_materialize       K2 diff expansion + K1 relocation + K3 rank patch
 *       fdy_members_download  HBM -> host copy of member images
 *       fdy_members_record    one member as the FNDG record the reference PrepareFn
 *                             returns (encode_graph_record, graph_model.cpp:205-218)
 *       fdy_load_members      the PrepareFn replacement for a whole archive:
 *                             integrity + fused kernel, result kept in HBM
 *                             (pipeline.cpp:411-417 + :506-514)
 *       fdy_crc64_segments    CRC-64/XZ of byte ranges, computed on the GPU
 *       fdy_sync, fdy_last_error
 *
 * Return codes: 0 on success, otherwise 1 + the reference Errc value
 * (errors.hpp:9-23: 1 invalid-argument ... 13 schema-violation), plus
 * FDY_ERR_CUDA and FDY_ERR_NO_DEVICE. fdy_last_error() returns the message of
 * the calling thread's last failure, formatted like foundry::Error::what()
 * ("<code-name>: <step>: <detail>").
 */
#ifndef FOUNDRY_B200_H
#define FOUNDRY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    FDY_OK = 0,
    FDY_ERR_INVALID_ARGUMENT = 1,
    FDY_ERR_SPEC_VIOLATION = 2,
    FDY_ERR_BINARY_FORMAT = 3,
    FDY_ERR_UNRESOLVED_KERNEL = 4,
    FDY_ERR_UNMAPPED_ADDRESS = 5,
    FDY_ERR_TOPOLOGY_MISMATCH = 6,
    FDY_ERR_LAYOUT_DIVERGENCE = 7,
    FDY_ERR_ARCHIVE_CORRUPTION = 8,
    FDY_ERR_OUT_OF_REGION = 9,
    FDY_ERR_UNKNOWN_ADDRESS = 10,
    FDY_ERR_DEVICE_STATE_UNINITIALIZED = 11,
    FDY_ERR_UNPATCHABLE_COMM = 12,
    FDY_ERR_SCHEMA_VIOLATION = 13,
    FDY_ERR_CUDA = 14,
    FDY_ERR_NO_DEVICE = 15,
};

typedef struct fdy_device fdy_device;
typedef struct fdy_store fdy_store;
typedef struct fdy_members fdy_members;
typedef struct fdy_serving fdy_serving;

/* ---------------------------------------------------------------- misc */
const char* fdy_last_error(void);
const char* fdy_version(void);
int fdy_device_count(void);

/* ---------------------------------------------------------------- kernel API */
int fdy_device_open(int ordinal, fdy_device** out);
void fdy_device_close(fdy_device* dev);
int fdy_sync(fdy_device* dev);

/* Copies `bytes` of an FNDT template store (foundry/store_format.h) into HBM. */
int fdy_store_upload(fdy_device* dev, const void* host_blob, size_t bytes, fdy_store** out);
/* Copies a resident store to another device (peer copy over NVLink when the
 * devices can access each other; staged otherwise). */
int fdy_store_fanout(const fdy_store* src, fdy_device* dst_dev, fdy_store** out);
/* Cross-process fan-out (one process per GPU): the owner exports a CUDA IPC
 * handle of its resident store; a peer process imports it, which pulls the
 * bytes GPU->GPU (NVLink P2P) into its own HBM and closes the mapping. */
int fdy_store_export(const fdy_store* store, unsigned char handle[64], uint64_t* bytes);
int fdy_store_import(fdy_device* dev, const unsigned char handle[64], uint64_t bytes,
                     fdy_store** out);
/* Pipelined chain fan-out (SURVEY §8(e) option ii), one process: dsts[0]
 * pulls the store from src chunk by chunk, dsts[i] from dsts[i-1] as each
 * chunk lands on it (per-chunk events, peer copies over NVLink), so the store
 * crosses each link once instead of src's egress carrying n copies.
 * chunk_bytes 0 = 2 MiB. outs[i] receives dsts[i]'s store. */
int fdy_store_fanout_chain(const fdy_store* src, fdy_device* const* dsts, uint32_t n, uint64_t chunk_bytes,
                           fdy_store** outs);
/* The same across processes (one per GPU): every link creates its buffer and
 * exports its handle (fdy_chain_create), the handles are exchanged (any
 * plumbing), then the head seeds from host memory and every other link pulls
 * from its predecessor; chunk k moves as soon as the predecessor published it
 * (a progress word in the predecessor's HBM, polled by the GPU: no host round
 * trip per chunk). fdy_chain_finish waits and returns the store; keep it alive
 * until the next link has finished (a barrier). */
typedef struct fdy_chain fdy_chain;
int fdy_chain_create(fdy_device* dev, uint64_t bytes, uint64_t chunk_bytes, fdy_chain** out,
                     unsigned char handle[64]);
int fdy_chain_seed(fdy_chain* chain, const void* host_blob);
int fdy_chain_pull(fdy_chain* chain, const unsigned char upstream[64]);
int fdy_chain_finish(fdy_chain* chain, fdy_store** out);
void fdy_chain_free(fdy_chain* chain);
void fdy_store_free(fdy_store* store);
size_t fdy_store_members_bytes(const fdy_store* store);

typedef struct {
    uint32_t rank;
    uint32_t world;
    uint64_t new_base;        /* 0: keep the captured VA base (no relocation) */
    const uint64_t* values;   /* optional per-rank value table (comm handles, peer buffers) */
    uint32_t n_values;
    int32_t grid;             /* 0: persistent grid = SMs x resident CTAs */
} fdy_materialize_desc;

/* Launches the fused materialization on the device stream. kernel_ms (may be
 * NULL) receives the kernel's CUDA-event duration (this call then blocks). */
int fdy_materialize(fdy_device* dev, const fdy_store* store, const fdy_materialize_desc* desc,
                    fdy_members** out, float* kernel_ms);
/* Reuses an existing output arena (same store) instead of allocating. */
int fdy_materialize_into(fdy_device* dev, const fdy_store* store,
                         const fdy_materialize_desc* desc, fdy_members* members,
                         float* kernel_ms);
/* Measurement variant of fdy_materialize_into: the template relocation grid and
 * the member pass run as separate launches and are timed separately (CUDA
 * events on the device stream; blocks). Same output. */
int fdy_materialize_timed_split(fdy_device* dev, const fdy_store* store, const fdy_materialize_desc* desc,
                                fdy_members* members, float* reloc_ms, float* member_ms);
/* Measurement only (bench.py's roofline): overwrites the arena with a plain
 * st.global.v4 fill and returns its CUDA-event duration — the floor a kernel
 * writing this many bytes reaches on this GPU. The arena holds no member
 * images afterwards. */
int fdy_members_write_probe(fdy_members* members, float* ms);
size_t fdy_members_bytes(const fdy_members* members);
int fdy_members_download(fdy_members* members, void* host_dst, size_t offset, size_t bytes);
void fdy_members_free(fdy_members* members);
/* One member graph of a materialized set as the FNDG record the reference's
 * encode_graph_record writes (graph_model.cpp:205-218) — i.e. what the
 * reference PrepareFn returns for `label` (pipeline.cpp:506-514), ready for its
 * own parse_graph_at(record, GraphLocator{label, 0, *len, *crc})
 * (graph_model.cpp:295-303). *len (and *crc, the record's CRC-64/XZ) are always
 * set; the bytes are written only when cap >= *len (query with buf NULL, then
 * copy: the second call reuses the first decode). invalid-argument for a label
 * outside the set. Thread-safe per call (prepare lanes may call concurrently). */
int fdy_members_record(fdy_members* members, uint32_t label, unsigned char* buf, size_t cap,
                       size_t* len, uint64_t* crc);


/* CRC-64/XZ of n byte ranges of a host buffer, computed on the GPU after one
 * H2D copy (ranges need not be aligned). digests receives n values. */
int fdy_crc64_segments(fdy_device* dev, const void* host, size_t bytes,
                       const uint64_t* offsets, const uint64_t* lengths, uint32_t n,
                       uint64_t* digests, float* kernel_ms);

/* The whole materialization path in one call — the GPU-native replacement of
 * the reference's verify_archive_integrity (pipeline.cpp:411-417) followed by
 * the PrepareFn over every member (pipeline.cpp:506-514): the template store
 * -> pinned staging -> HBM with a GPU CRC of each piece as it lands -> fused
 * K2+K1+K3 for desc->(rank, world, new_base) -> member images (store_format.h
 * layout) copied to host_out; meanwhile every other archive file is CRCed on
 * the host (`lanes` threads at the lowest CPU priority; the store uses up to 4
 * lanes at normal priority) and all digests are checked against the manifest
 * before the call returns. host_out may be NULL (images stay in HBM only);
 * out_len receives the image bytes. */
typedef struct {
    double total_ms, read_ms, integrity_ms, materialize_ms, d2h_ms;
    float crc_kernel_ms, kernel_ms;
    uint64_t h2d_bytes, d2h_bytes, member_bytes, graphs, nodes;
} fdy_prepare_timings;

int fdy_prepare_archive(fdy_device* dev, const char* archive, const fdy_materialize_desc* desc,
                        uint32_t lanes, void* host_out, size_t cap, size_t* out_len,
                        fdy_prepare_timings* timings);
/* The GPU PrepareFn in one call, result kept in HBM: the archive's files are
 * staged and integrity-checked (GPU CRC of the store, host CRC of the rest,
 * verify_archive_integrity pipeline.cpp:411-417), the fused K2+K1+K3 kernel
 * materializes every member for desc, and the returned fdy_members serves
 * fdy_members_record / fdy_members_download. A reference-written archive (no
 * templates.fdt) is packed on the host first. */
int fdy_load_members(fdy_device* dev, const char* archive, const fdy_materialize_desc* desc, uint32_t lanes,
                     fdy_members** out, fdy_prepare_timings* timings);

/* Pinned host memory usable as host_out (released with fdy_host_free). */
void* fdy_host_alloc(fdy_device* dev, size_t bytes);
void fdy_host_free(void* p);

/* ---------------------------------------------------------------- session API */
typedef struct {
    uint32_t rank;           /* LoadOptions.rank */
    uint32_t world;          /* LoadOptions.world */
    int32_t preallocate;     /* LoadOptions.preallocate (bool) */
    uint32_t prepare_lanes;  /* LoadOptions.prepare_lanes: host threads for file staging */
    int32_t device;          /* B200: CUDA device ordinal */
    int32_t relocate;        /* B200: rebase embedded addresses if the VA region moves */
    /* FaultInjection (pipeline.hpp:73-78) */
    int32_t skip_binary_restore;
    int32_t skip_device_init;
    int64_t base_shift_granules;
    int32_t extra_prewindow_alloc;
    int32_t share_execs;     /* B200: one instantiated exec per graph shape (LoadOptions.share_execs) */
    int32_t device_updates;  /* B200: serve applies kernel-node parameters from the GPU (LoadOptions.device_updates) */
    /* B200: this rank's value table for the archive's comm slots (comm_slots.bin:
     * comm handles, peer buffer addresses; LoadOptions.comm_values) */
    const uint64_t* comm_values;
    uint32_t n_comm_values;
} fdy_load_options;

void fdy_load_options_init(fdy_load_options* opts);
int fdy_load(const char* archive, const fdy_load_options* opts, fdy_serving** out);
int fdy_serving_replay(fdy_serving* s, uint32_t batch, char* buf, size_t cap, size_t* len);
int fdy_serving_batches(fdy_serving* s, uint32_t* out, size_t cap, size_t* count);
int fdy_serving_counter(fdy_serving* s, const char* key, uint64_t* value);
/* "key=value\n" lines, sorted by key. */
int fdy_serving_counters(fdy_serving* s, char* buf, size_t cap, size_t* len);
uint32_t fdy_serving_template_count(const fdy_serving* s);
void fdy_serving_close(fdy_serving* s);
/* Bytes written to buf (up to cap); *len = the record's full length. */
int fdy_serving_capture_graph(fdy_serving* s, uint32_t batch, unsigned char* buf, size_t cap, size_t* len);
/* GPU-side SAVE to an archive directory (reference SAVE
 * pipeline.cpp:249-405): every batch stream-captured on the device and
 * extracted, comm nodes lowered back to stubs (rank_forge.cpp:132-152
 * inverted), grouped (templater.cpp:18-52), serialized (graph_model.cpp:244-269)
 * and written with the catalog, memory log, patch table, binaries and a packed
 * templates.fdt. The archive loads in the reference and here. */
int fdy_serving_save_captured(fdy_serving* s, const char* out_dir);

#ifdef __cplusplus
}
#endif
#endif
