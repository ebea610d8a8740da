/* foundry_oracle.h — CPU restatement of the reference's LOAD-side per-member
 * work (TEST INFRASTRUCTURE, never linked by the product; see oracle/README.md).
 *
 * Every entry point names the reference function it restates. Parity of this
 * restatement with the reference itself is pinned by tests/test_oracle.py:
 * CRC KATs (test_hash.cpp:13-27), and byte-identical containers against
 * oracle/_ref/ref_tool `prepare` (the reference PrepareFn) on every member
 * of every tier-R workload; relocation (delta != 0, no reference function) is
 * pinned by replaying our relocated members on the reference simulated driver
 * at the shifted base (ref_tool `replay`), whose hidden offsets are the
 * ground truth for which slots are device addresses.
 */
#ifndef FOUNDRY_ORACLE_H
#define FOUNDRY_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes: the reference Errc values (errors.hpp:9-23) + 1; 0 = ok. */
enum {
    FO_OK = 0,
    FO_INVALID_ARGUMENT = 1,
    FO_BINARY_FORMAT = 3,
    FO_UNRESOLVED_KERNEL = 4,
    FO_ARCHIVE_CORRUPTION = 8,
};

/* CRC-64/XZ, table-driven byte at a time: hash.cpp:13-25,53-69. */
uint64_t fo_crc64(const uint8_t* data, size_t len);
/* Bitwise CRC-64/XZ, no table: the reference test oracle support.hpp:45-55. */
uint64_t fo_crc64_bitwise(const uint8_t* data, size_t len);

/* Number of records in an FNDG container (graph_model.cpp:271-293); -code on error. */
int64_t fo_graph_count(const uint8_t* graphs, size_t len);

/* Materializes every member of graphs.bin for one rank and returns the
 * result as an FNDG container (serialize_graphs layout, graph_model.cpp:244-269)
 * in locator order. Per member, exactly the reference PrepareFn
 * (pipeline.cpp:506-514): parse_graph_at (graph_model.cpp:295-303: record CRC,
 * decode_graph_record :220-240, validate :41-64, label check) followed by
 * relocation (SURVEY.md §8c rule; identity when new_base == old_base) and
 * apply_rank_patches (rank_forge.cpp:132-152) when patch.bin has entries for
 * the label. Members are processed by `lanes` worker threads, one member per
 * task, like the reference prepare lanes (templater.cpp:102-130).
 *
 * Relocation rule: every 8-byte-aligned u64 slot (o % 8 == 0, o + 8 <= len)
 * of every kernel argument buffer, plus memcpy src/dst and memset dst, whose
 * value v lies in [old_base, old_base + final_offset) becomes v + (new_base -
 * old_base). Order: relocate, then rank-patch.
 *
 * On success *out receives a malloc'd buffer (release with fo_free) of
 * *out_len bytes. Returns 0 or an error code; on error err_msg (if non-NULL,
 * err_cap bytes) receives a reference-style message. n_relocated (may be
 * NULL) receives the number of rewritten slots. */
int fo_materialize_container(const uint8_t* graphs, size_t graphs_len,
                             const uint8_t* patch, size_t patch_len,
                             uint64_t real_comm_hash, uint32_t rank, uint32_t world,
                             uint64_t old_base, uint64_t final_offset, uint64_t new_base,
                             unsigned lanes, uint8_t** out, size_t* out_len,
                             uint64_t* n_relocated, char* err_msg, size_t err_cap);

/* The same with the archive's comm slots (comm_slots.bin; slots/slots_len
 * 0 = none) applied after apply_rank_patches from the rank's value table
 * (values[n_values]). Slot rule: archive.hpp CommSlot. */
int fo_materialize_container_ex(const uint8_t* graphs, size_t graphs_len,
                                const uint8_t* patch, size_t patch_len,
                                const uint8_t* slots, size_t slots_len,
                                const uint64_t* values, uint32_t n_values,
                                uint64_t real_comm_hash, uint32_t rank, uint32_t world,
                                uint64_t old_base, uint64_t final_offset, uint64_t new_base,
                                unsigned lanes, uint8_t** out, size_t* out_len,
                                uint64_t* n_relocated, char* err_msg, size_t err_cap);

void fo_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
