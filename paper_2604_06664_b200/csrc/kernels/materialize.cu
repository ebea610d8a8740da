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
    uint8_t ometa[FDT_TILE_CHUNKS];     // relocation-meta overrides from diff entries (0x80 | lanes)
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

// Expands 4 mask bits into a 32-bit byte-select word (bit i -> byte i = 0xFF).
__device__ __forceinline__ uint32_t byte_select(uint32_t m4) {
    return ((m4 * 0x00204081u) & 0x01010101u) * 0xFFu;
}

__device__ __forceinline__ uint4 merge_bytes(uint4 base, uint4 over, uint32_t mask) {
    const uint32_t s0 = byte_select(mask & 0xFu), s1 = byte_select((mask >> 4) & 0xFu);
    const uint32_t s2 = byte_select((mask >> 8) & 0xFu), s3 = byte_select((mask >> 12) & 0xFu);
    return make_uint4((base.x & ~s0) | (over.x & s0), (base.y & ~s1) | (over.y & s1),
                      (base.z & ~s2) | (over.z & s2), (base.w & ~s3) | (over.w & s3));
}

// 16-byte little-endian image of `value` placed so that byte j of the chunk
// holds value byte (j - shift); bytes outside the value are zero.
__device__ __forceinline__ uint4 place_value(uint64_t value, int shift) {
    uint64_t lo, hi;
    if (shift >= 0) {
        const int s = 8 * shift;
        lo = s < 64 ? value << s : 0ull;
        hi = s == 0 ? 0ull : (s < 64 ? value >> (64 - s) : value << (s - 64));
    } else {
        lo = value >> (-8 * shift);
        hi = 0ull;
    }
    return make_uint4(uint32_t(lo), uint32_t(lo >> 32), uint32_t(hi), uint32_t(hi >> 32));
}

__device__ __forceinline__ uint64_t rank_op_value(const fdt_rank_op& op, const FdyMaterializeArgs& a) {
    switch (op.kind) {
        case FDT_ROP_RANK: return a.rank;
        case FDT_ROP_WORLD: return a.world;
        case FDT_ROP_KERNEL: return op.aux;
        default: return op.aux < a.n_values ? a.values[op.aux] : 0ull;
    }
}

__device__ __forceinline__ void relocate_pair(uint32_t& lo, uint32_t& hi, bool flagged,
                                              const FdyMaterializeArgs& a) {
    const uint64_t x = (uint64_t(hi) << 32) | lo;
    const uint64_t y = (flagged && x - a.old_base < a.span) ? x + a.delta : x;
    lo = uint32_t(y);
    hi = uint32_t(y >> 32);
}

// Phases per tile, each convergent across the CTA:
//   B  diff-parallel: one thread per diff entry overlays its chunk in smem
//   C  chunk-parallel relocation (skipped when delta == 0, a uniform branch)
//   D  op-run-parallel rank patch: one thread per chunk's run of ops
__global__ void __launch_bounds__(kThreads)
fdy_materialize_kernel(const FdyMaterializeArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x;
    const bool relocating = a.delta != 0ull;

    if (tid == 0) {
        mbar_init(&s.bar[0], 1);
        mbar_init(&s.bar[1], 1);
        fence_mbar_init();
    }
    for (int i = tid; i < FDT_TILE_CHUNKS; i += kThreads) s.ometa[i] = 0;
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
        // prefetch the next tile into the other stage once its store has drained
        if (tid == 0 && next < a.n_tiles) {
            bulk_wait_reads();
            const fdt_tile& N = a.tiles[next];
            mbar_expect_tx(&s.bar[stage ^ 1], N.nchunks * 16u);
            bulk_load(s.buf[stage ^ 1], a.store + N.src_off, N.nchunks * 16u, &s.bar[stage ^ 1]);
        }
        uint4* buf = s.buf[stage];
        mbar_wait(&s.bar[stage], (parity >> stage) & 1u);
        parity ^= 1u << stage;

        // B: K2 diff overlay
        for (uint32_t e = T.diff_lo + tid; e < T.diff_hi; e += kThreads) {
            const uint32_t c = __ldg(a.didx + e) - T.chunk_base;
            const uint32_t dm = __ldg(a.dmeta + e);
            buf[c] = merge_bytes(buf[c], __ldg(a.ddata + e), dm & FDT_DMETA_MASK);
            if (relocating && (dm & FDT_DMETA_RELOC_OVERRIDE))
                s.ometa[c] = static_cast<uint8_t>(0x80u | ((dm >> FDT_DMETA_RELOC_SHIFT) & 3u));
        }
        __syncthreads();

        // C: K1 relocation of flagged lanes whose value lies in the captured range
        if (relocating) {
            const uint8_t* meta = a.cmeta + (T.src_off - a.timage_base) / 16;
            for (uint32_t c = tid; c < T.nchunks; c += kThreads) {
                uint32_t m = __ldg(meta + c);
                const uint32_t o = s.ometa[c];
                if (o) {
                    m = o & 3u;
                    s.ometa[c] = 0;
                }
                if (m) {
                    uint4 v = buf[c];
                    relocate_pair(v.x, v.y, m & FDT_CMETA_LANE0, a);
                    relocate_pair(v.z, v.w, m & FDT_CMETA_LANE1, a);
                    buf[c] = v;
                }
            }
            __syncthreads();
        }

        // D: K3 rank ops; ops on one chunk are applied in table order by one thread
        for (uint32_t i = T.rop_lo + tid; i < T.rop_hi; i += kThreads) {
            const uint32_t ch = a.rops[i].chunk;
            if (i != T.rop_lo && a.rops[i - 1].chunk == ch) continue;
            uint4 v = buf[ch - T.chunk_base];
            for (uint32_t j = i; j < T.rop_hi; ++j) {
                const fdt_rank_op op = a.rops[j];
                if (op.chunk != ch) break;
                v = merge_bytes(v, place_value(rank_op_value(op, a), op.shift), op.mask);
            }
            buf[ch - T.chunk_base] = v;
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) bulk_store(a.out + T.dst_off, buf, T.nchunks * 16u);
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
