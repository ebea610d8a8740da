// Device body shared by every generated trace kernel (ABI: foundry/trace_abi.h).
// Compiled once to PTX (-rdc) at build time; the packer links it into one
// cubin per cataloged binary next to thin .entry wrappers that pass their
// parameter block (cvta.param) plus the entry's baked-in hidden offsets.
#include <cstdint>

#include "foundry/trace_abi.h"

extern "C" {
__device__ fdy_trace_ctx* fdy_trace_context;  // set per library by the host
__device__ unsigned int fdy_device_inited;     // set by run_device_init
}

extern "C" __device__ __noinline__ void fdy_trace_body(const unsigned char* args, unsigned int n,
                                                       const unsigned int* hidden, unsigned int nh,
                                                       unsigned int entry_id,
                                                       unsigned int needs_init) {
    if ((blockIdx.x | blockIdx.y | blockIdx.z | threadIdx.x | threadIdx.y | threadIdx.z) != 0) return;
    fdy_trace_ctx* ctx = fdy_trace_context;
    if (ctx == nullptr) return;
    const unsigned long long bytes = FDY_TRACE_HEADER_BYTES + ((n + 15u) & ~15u);
    const unsigned long long at = atomicAdd(ctx->cursor, bytes);
    if (at + bytes > ctx->capacity) return;
    unsigned char* rec = ctx->arena + at;
    unsigned char* body = rec + FDY_TRACE_HEADER_BYTES;
    // the parameter block is 8-byte aligned (.param .align 8)
    unsigned int i = 0;
#pragma unroll 1
    for (; i + 8 <= n; i += 8)
        *reinterpret_cast<unsigned long long*>(body + i) =
            *reinterpret_cast<const unsigned long long*>(args + i);
#pragma unroll 1
    for (; i < n; ++i) body[i] = args[i];
    unsigned int flags = 0;
#pragma unroll 1
    for (unsigned int h = 0; h < nh; ++h) {
        unsigned long long a = 0;
#pragma unroll 1
        for (int k = 7; k >= 0; --k) a = (a << 8) | args[hidden[h] + k];
        const unsigned long long g = (a - ctx->map_base) >> ctx->granule_shift;
        const bool mapped = a >= ctx->map_base && g < ctx->map_granules &&
                            ((ctx->bitmap[g >> 6] >> (g & 63)) & 1ull);
        if (mapped) atomicAdd(reinterpret_cast<unsigned long long*>(a & ~7ull), 1ull);
        else flags |= FDY_TRACE_FLAG_UNMAPPED;
    }
    if (needs_init && !fdy_device_inited) flags |= FDY_TRACE_FLAG_UNINIT;
    unsigned int smem;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(smem));
    fdy_trace_header* hd = reinterpret_cast<fdy_trace_header*>(rec);
    hd->entry_id = entry_id;
    hd->n_bytes = n;
    hd->flags = flags;
    hd->dyn_smem = smem;
    hd->grid[0] = gridDim.x;
    hd->grid[1] = gridDim.y;
    hd->grid[2] = gridDim.z;
    hd->block[0] = blockDim.x;
    hd->block[1] = blockDim.y;
    hd->block[2] = blockDim.z;
    __threadfence();
    hd->magic = FDY_TRACE_MAGIC;
}
