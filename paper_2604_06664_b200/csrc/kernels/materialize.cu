// Fused graph-set materialization for sm_100a: K2 (template diff expansion)
// -> K1 (VA relocation) -> K3 (rank / comm-state patch), one pass over HBM.
//
// Work unit: a tile = up to FDT_TILE_CHUNKS (1024) 16-byte chunks of one
// member image (layout: foundry/store_format.h). Each persistent CTA walks the
// tile list with a 2-stage TMA bulk-copy pipeline:
//
//   cp.async.bulk  global -> smem   template chunk tile (mbarrier complete_tx)
//   overlay        diff chunks (byte masks) from the member's diff stream
//   relocate       8-byte lanes flagged by the chunk meta whose value lies in
//                  [old_base, old_base + span): v += delta
//   patch          the tile's rank ops (rank/world u64, stub->real kernel
//                  index, per-rank value table) on the smem tile
//   cp.async.bulk  smem -> global   member image tile (bulk_group)
//
// The reference does this work per node on CPU prepare lanes: parse_graph_at
// (graph_model.cpp:295-303) + apply_rank_patches (rank_forge.cpp:132-152);
// relocation has no reference function (SURVEY.md §8c rule). Pure integer
// streaming: no tensor-core work exists here, the bound is HBM bandwidth.
#include <cstdint>

#include "foundry/store_format.h"
#include "fdy_kernels.h"

namespace {

constexpr int kThreads = 256;
constexpr int kChunksPerThread = FDT_TILE_CHUNKS / kThreads;
static_assert(FDT_TILE_CHUNKS % kThreads == 0, "tile must split evenly across the CTA");

struct __align__(128) Smem {
    uint4 buf[2][FDT_TILE_CHUNKS];      // 2 x 16 KiB stages
    unsigned long long bar[2];          // mbarriers, one per stage
    uint16_t slot[FDT_TILE_CHUNKS];     // chunk -> 1 + diff entry offset (0 = none)
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "FDY_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra FDY_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes,
                                          unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_addr(dst_smem)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_addr(src_smem)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_reads() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint64_t relocate_lane(uint64_t v, const FdyMaterializeArgs& a) {
    return (v - a.old_base < a.span) ? v + a.delta : v;
}

__device__ __forceinline__ uint4 merge_bytes(uint4 base, uint4 over, uint32_t mask) {
    // expand a 16-bit byte mask into four 32-bit lane selectors
    uint32_t w[4] = {base.x, base.y, base.z, base.w};
    const uint32_t o[4] = {over.x, over.y, over.z, over.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t m4 = (mask >> (4 * i)) & 0xFu;
        // byte-select mask: 0x000000FF per set bit
        const uint32_t sel = ((m4 & 1u) ? 0x000000FFu : 0u) | ((m4 & 2u) ? 0x0000FF00u : 0u) |
                             ((m4 & 4u) ? 0x00FF0000u : 0u) | ((m4 & 8u) ? 0xFF000000u : 0u);
        w[i] = (w[i] & ~sel) | (o[i] & sel);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void __launch_bounds__(kThreads)
fdy_materialize_kernel(const FdyMaterializeArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x;

    if (tid == 0) {
        mbar_init(&s.bar[0], 1);
        mbar_init(&s.bar[1], 1);
        fence_mbar_init();
    }
    for (int i = tid; i < FDT_TILE_CHUNKS; i += kThreads) s.slot[i] = 0;
    __syncthreads();

    uint32_t t = blockIdx.x;
    if (t >= a.n_tiles) return;
    if (tid == 0) {
        const fdt_tile& first = a.tiles[t];
        mbar_expect_tx(&s.bar[0], first.nchunks * 16u);
        bulk_load(s.buf[0], a.store + first.src_off, first.nchunks * 16u, &s.bar[0]);
    }

    uint32_t stage = 0;
    uint32_t parity = 0u;  // bit s = expected phase parity of stage s
    for (; t < a.n_tiles; t += gridDim.x) {
        const fdt_tile T = a.tiles[t];
        const uint32_t next = t + gridDim.x;

        // K2 index: scatter this tile's diff entries into the chunk slot map
        for (uint32_t e = T.diff_lo + tid; e < T.diff_hi; e += kThreads)
            s.slot[a.didx[e] - T.chunk_base] = static_cast<uint16_t>(e - T.diff_lo + 1);

        // prefetch the next tile into the other stage once its store has drained
        if (tid == 0 && next < a.n_tiles) {
            bulk_wait_reads();
            const fdt_tile& N = a.tiles[next];
            mbar_expect_tx(&s.bar[stage ^ 1], N.nchunks * 16u);
            bulk_load(s.buf[stage ^ 1], a.store + N.src_off, N.nchunks * 16u, &s.bar[stage ^ 1]);
        }
        __syncthreads();
        mbar_wait(&s.bar[stage], (parity >> stage) & 1u);
        parity ^= 1u << stage;

        const uint8_t* meta = a.cmeta + (T.src_off - a.timage_base) / 16;
#pragma unroll
        for (int k = 0; k < kChunksPerThread; ++k) {
            const uint32_t c = tid + k * kThreads;
            if (c >= T.nchunks) break;
            uint4 v = s.buf[stage][c];
            uint32_t m = meta[c];
            const uint32_t sl = s.slot[c];
            if (sl) {  // K2: overlay the member's bytes
                const uint32_t e = T.diff_lo + sl - 1;
                const uint32_t dm = __ldg(a.dmeta + e);
                const uint4 d = __ldg(a.ddata + e);
                v = merge_bytes(v, d, dm & FDT_DMETA_MASK);
                if (dm & FDT_DMETA_RELOC_OVERRIDE) m = (dm >> FDT_DMETA_RELOC_SHIFT) & 3u;
                s.slot[c] = 0;
            }
            if (m) {  // K1: relocate flagged lanes whose value is in the captured range
                if (m & FDT_CMETA_LANE0) {
                    uint64_t x = (uint64_t(v.y) << 32) | v.x;
                    x = relocate_lane(x, a);
                    v.x = uint32_t(x);
                    v.y = uint32_t(x >> 32);
                }
                if (m & FDT_CMETA_LANE1) {
                    uint64_t x = (uint64_t(v.w) << 32) | v.z;
                    x = relocate_lane(x, a);
                    v.z = uint32_t(x);
                    v.w = uint32_t(x >> 32);
                }
            }
            s.buf[stage][c] = v;
        }
        __syncthreads();

        // K3: rank ops, in table order (ops on one chunk may overlap)
        if (tid == 0) {
            unsigned char* tile_bytes = reinterpret_cast<unsigned char*>(s.buf[stage]);
            for (uint32_t i = T.rop_lo; i < T.rop_hi; ++i) {
                const fdt_rank_op op = a.rops[i];
                uint64_t value;
                switch (op.kind) {
                    case FDT_ROP_RANK: value = a.rank; break;
                    case FDT_ROP_WORLD: value = a.world; break;
                    case FDT_ROP_KERNEL: value = op.aux; break;
                    default: value = op.aux < a.n_values ? a.values[op.aux] : 0ull; break;
                }
                unsigned char* chunk = tile_bytes + 16u * (op.chunk - T.chunk_base);
                for (int j = 0; j < 16; ++j)
                    if (op.mask & (1u << j)) chunk[j] = static_cast<unsigned char>(value >> (8 * (j - op.shift)));
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) bulk_store(a.out + T.dst_off, s.buf[stage], T.nchunks * 16u);
        stage ^= 1u;
    }
    if (tid == 0) bulk_wait_all();
}

}  // namespace

extern "C" size_t fdy_materialize_smem_bytes() { return sizeof(Smem); }

extern "C" cudaError_t fdy_launch_materialize(const FdyMaterializeArgs* args, int grid,
                                              cudaStream_t stream) {
    if (args->n_tiles == 0) return cudaSuccess;
    // per-device attribute; cheap enough to set on every launch
    const cudaError_t e = cudaFuncSetAttribute(
        fdy_materialize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(Smem)));
    if (e != cudaSuccess) return e;
    fdy_materialize_kernel<<<grid, kThreads, sizeof(Smem), stream>>>(*args);
    return cudaGetLastError();
}

extern "C" cudaError_t fdy_materialize_occupancy(int* blocks_per_sm) {
    cudaError_t e = cudaFuncSetAttribute(fdy_materialize_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(sizeof(Smem)));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fdy_materialize_kernel,
                                                         kThreads, sizeof(Smem));
}
