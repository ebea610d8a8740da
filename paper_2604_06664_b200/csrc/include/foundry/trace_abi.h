/* trace_abi.h — device/host ABI of the replay-verification trace kernels.
 *
 * Every cataloged kernel entrypoint is re-materialized as a real sm_100a
 * function with the exact reference name and argument-buffer size; its body
 * (kernels/trace_body.cu) is the on-device half of the reference replay check
 * (sim_driver.cpp:402-479): it appends one record per launch holding the launch
 * geometry and the exact parameter bytes the kernel received, dereferences the
 * entry's hidden pointer offsets (only when the logical mapping bitmap says the
 * granule is mapped, so a bad pointer never faults the context) and checks the
 * module's device-init state. The host matches records to graph nodes and
 * renders the reference LaunchTrace text from them.
 */
#ifndef FOUNDRY_TRACE_ABI_H
#define FOUNDRY_TRACE_ABI_H

#include <stdint.h>

#define FDY_TRACE_FLAG_UNMAPPED 0x1u
#define FDY_TRACE_FLAG_UNINIT 0x2u
#define FDY_TRACE_HEADER_BYTES 64u

typedef struct {
    uint32_t entry_id; /* (binary ordinal << 16) | entrypoint index */
    uint32_t n_bytes;  /* parameter bytes that follow the header */
    uint32_t flags;
    uint32_t dyn_smem;
    uint32_t grid[3];
    uint32_t block[3];
    uint32_t magic; /* 0xFD7EACE5 once the record is complete */
    uint32_t pad[5];
} fdy_trace_header; /* 64 bytes, then round_up(n_bytes, 16) parameter bytes */

#define FDY_TRACE_MAGIC 0xFD7EACE5u

typedef struct {
    unsigned char* arena;
    unsigned long long* cursor; /* bytes used */
    uint64_t capacity;
    const uint64_t* bitmap; /* one bit per granule of the logical region */
    uint64_t map_base;
    uint64_t map_granules;
    uint32_t granule_shift;
    uint32_t pad;
} fdy_trace_ctx;

#endif
