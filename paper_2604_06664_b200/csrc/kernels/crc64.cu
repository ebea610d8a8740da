// GPU CRC-64/XZ for archive integrity: replaces the
// reference's single-threaded byte-at-a-time walk over every archive file
// (verify_archive_integrity, pipeline.cpp:411-417; Crc64::update, hash.cpp:53-61)
// with an HBM-resident, chunk-parallel computation.
//
// Algebra. Let F be the linear part of the CRC (init 0, no final xor, the
// reflected bit order of hash.cpp) and A_k "advance by k bytes", i.e.
// multiplication by x^(8k) mod P. Then for CRC-64/XZ (init = xorout = ~0)
//     F(A || B) = A_|B|(F(A)) ^ F(B)
//     crc(M)    = ~(F(M) ^ A_|M|(~0))
// Every combine below multiplies by a CONSTANT power of x, and
// multiplication by a constant is a 64x64 GF(2) linear map: 16 nibble
// tables of 16 entries (2 KB) in shared memory, one lookup per nibble. A
// table is 128 B = all 32 banks, so a warp's lookups never conflict.
//
//   crc_blocks_kernel  persistent CTAs (tables built once per CTA). Per 64 KiB
//                      block each thread runs the nibble-sliced CRC over its
//                      256 contiguous bytes; the CTA combines the 256 pieces
//                      with a tree whose level-L multiplier is A_(256 * 2^L)
//                      (5 levels of warp shuffles, 3 across warps).
//   crc_fold_kernel    one CTA per segment: Horner per thread over a run of
//                      full blocks, then the same kind of tree across threads
//                      (multipliers A_(65536 * run * 2^L)), then the last
//                      block and the init/xorout term.
// A short block (a segment's last) takes the generic path: per-thread
// mulmod by x^(8 * bytes after the piece), then a plain XOR reduction.
#include <algorithm>
#include <cstdint>

#include "fdy_kernels.h"

namespace {

constexpr uint64_t kPoly = 0xC96C5795D7870F42ull;
constexpr int kThreads = 256;
constexpr uint32_t kBytesPerThread = kCrcBlockBytes / kThreads;
static_assert(kBytesPerThread == 256 && kCrcBlockBytes == 65536, "braid/tree constants assume 8 warps x 8 KiB");
constexpr int kFoldThreads = 1024;
constexpr int kFoldLevels = 20;   // up to 2^20 blocks (64 GiB) per segment (k = 19..38)

__constant__ uint64_t c_x2k[64];  // x^(2^k) mod P, k = 0..63 (host-computed)

typedef uint64_t NibbleTable[16][16];

// Constant-multiplier tables, host-computed once per device (set_constants):
// g_tables[k - kFirstPow] multiplies by x^(2^k), k = 6..39. A_n = x^(8n):
//   k = 6  A_8      per-word slicing step          k = 12   A_512 braid step
//   k = 7..11       lane tree A_(16 * 2^L)         k = 16..18  warp tree A_(8192 * 2^L)
//   k = 19..38      segment tree A_(65536 * 2^L)
constexpr int kFirstPow = 6, kNumTables = 34;
constexpr int kBlockPows = 13;  // k = 6..18 live in the blocks kernel's shared memory
__device__ NibbleTable g_tables[kNumTables];

__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b) {
    uint64_t p = 0;
#pragma unroll 8
    for (int i = 63; i >= 0; --i) {
        if ((a >> i) & 1ull) p ^= b;
        b = (b & 1ull) ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
}

// x^(8 n) mod P
__device__ __forceinline__ uint64_t x8n(uint64_t n) {
    uint64_t p = 1ull << 63;
    for (int k = 3; n; n >>= 1, ++k)
        if (n & 1ull) p = mulmod(c_x2k[k & 63], p);
    return p;
}

// v * K mod P through K's nibble table
__device__ __forceinline__ uint64_t mulc(const NibbleTable& N, uint64_t v) {
    const uint32_t lo = uint32_t(v), hi = uint32_t(v >> 32);
    uint64_t r = N[0][lo & 0xF];
#pragma unroll
    for (int j = 1; j < 8; ++j) r ^= N[j][(lo >> (4 * j)) & 0xF];
#pragma unroll
    for (int j = 0; j < 8; ++j) r ^= N[8 + j][(hi >> (4 * j)) & 0xF];
    return r;
}

__device__ __forceinline__ uint64_t crc_byte_bitwise(uint64_t c, uint8_t byte) {
    c ^= byte;
#pragma unroll
    for (int b = 0; b < 8; ++b) c = (c & 1ull) ? (c >> 1) ^ kPoly : c >> 1;
    return c;
}

__device__ __forceinline__ uint64_t xor_reduce_warp(uint64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v ^= __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

// Ordered combine of 2^levels values held one per lane (lane 0 first):
// level L: left = A(left) ^ right, A = table L. Lane 0 ends with the result.
__device__ __forceinline__ uint64_t tree_warp(const NibbleTable* T, uint64_t v, int levels) {
    const int lane = threadIdx.x & 31;
    for (int L = 0; L < levels; ++L) {
        const uint64_t right = __shfl_down_sync(0xFFFFFFFFu, v, 1 << L);
        if ((lane & ((2 << L) - 1)) == 0) v = mulc(T[L], v) ^ right;
    }
    return v;
}

__global__ void __launch_bounds__(kThreads)
crc_blocks_kernel(const unsigned char* __restrict__ base, const FdyCrcBlock* __restrict__ blocks,
                  uint32_t n_blocks, uint64_t* __restrict__ out_crc, uint64_t* __restrict__ out_len) {
    __shared__ NibbleTable T[kBlockPows];  // T[k - 6]: multiply by x^(2^k)
    __shared__ uint64_t wpart[kThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const NibbleTable& A8 = T[6 - kFirstPow];
    const NibbleTable& A512 = T[12 - kFirstPow];

    {  // tables -> shared memory, once per persistent CTA (26 KB, L2-resident)
        const uint4* src = reinterpret_cast<const uint4*>(&g_tables[0]);
        uint4* dst = reinterpret_cast<uint4*>(&T[0]);
        for (int i = tid; i < int(sizeof(NibbleTable)) * kBlockPows / 16; i += kThreads) dst[i] = src[i];
    }
    __syncthreads();

    for (uint32_t b = blockIdx.x; b < n_blocks; b += gridDim.x) {
        const FdyCrcBlock blk = blocks[b];
        if (blk.length == kCrcBlockBytes && (blk.offset & 15u) == 0) {  // uniform per CTA
            // Braid: warp w owns the block's 8 KiB region w; lane l takes its
            // 16-byte chunks j = 32 k + l (each warp load is 512 contiguous
            // bytes) and runs Horner with the 512-byte advance:
            //   s_l = XOR_k A_512^(15-k) (A_8 w0_j ^ w1_j)
            // Region: F = A_8 * XOR_l A_16^(31-l) s_l (lane tree, then A_8).
            const uint4* p = reinterpret_cast<const uint4*>(base + blk.offset) + warp * 512 + lane;
            uint64_t c = 0;
#pragma unroll 4
            for (int k = 0; k < 16; ++k) {
                const uint4 v = __ldg(p + 32 * k);
                c = mulc(A512, c) ^ mulc(A8, (uint64_t(v.y) << 32) | v.x) ^ ((uint64_t(v.w) << 32) | v.z);
            }
            c = tree_warp(&T[7 - kFirstPow], c, 5);
            if (lane == 0) wpart[warp] = mulc(A8, c);
            __syncthreads();
            if (warp == 0) {  // 8 regions of 8 KiB
                c = tree_warp(&T[16 - kFirstPow], lane < kThreads / 32 ? wpart[lane] : 0ull, 3);
                if (lane == 0) {
                    out_crc[b] = c;
                    out_len[b] = blk.length;
                }
            }
        } else {  // a segment's short last block, or any block of a segment that is
                  // not 16-byte aligned (graph records inside graphs.bin): 256
                  // contiguous bytes per thread, weighted by generic mulmod,
                  // plain XOR reduction
            const uint32_t lo = umin(blk.length, tid * kBytesPerThread);
            const uint32_t hi = umin(blk.length, lo + kBytesPerThread);
            const unsigned char* p = base + blk.offset + lo;
            uint64_t c = 0;
            uint32_t i = 0;
            const uint32_t n = hi - lo;
            // bytewise up to the first 16-byte boundary (the linear CRC state
            // takes bytes and words alike)
            for (; i < n && (reinterpret_cast<uintptr_t>(p + i) & 15u); ++i) c = crc_byte_bitwise(c, p[i]);
            for (; i + 16 <= n; i += 16) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(p + i));
                c = mulc(A8, c ^ ((uint64_t(v.y) << 32) | v.x));
                c = mulc(A8, c ^ ((uint64_t(v.w) << 32) | v.z));
            }
            for (; i < n; ++i) c = crc_byte_bitwise(c, p[i]);
            if (n) c = mulmod(c, x8n(blk.length - hi));
            c = xor_reduce_warp(c);
            if (lane == 0) wpart[warp] = c;
            __syncthreads();
            if (tid == 0) {
                uint64_t f = 0;
#pragma unroll
                for (int w = 0; w < kThreads / 32; ++w) f ^= wpart[w];
                out_crc[b] = f;
                out_len[b] = blk.length;
            }
        }
        __syncthreads();  // wpart is reused by the next block
    }
}

// x^(8 n) mod P with one warp: lane i holds the factor of bit i (5 levels of
// generic mulmod instead of up to 32 in sequence). Result in every lane.
__device__ __forceinline__ uint64_t x8n_warp(uint64_t n) {
    const int lane = threadIdx.x & 31;
    uint64_t f = 1ull << 63;
    if (lane < 61 - 3 && ((n >> lane) & 1ull)) f = c_x2k[lane + 3];
    // bits 32..60 of n (segments > 4 GiB): fold them into lanes 0..28
    if (lane + 32 < 61 && ((n >> (lane + 32)) & 1ull)) f = mulmod(f, c_x2k[(lane + 35) & 63]);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const uint64_t g = __shfl_xor_sync(0xFFFFFFFFu, f, o);
        f = mulmod(f, g);
    }
    return f;
}

__global__ void __launch_bounds__(kFoldThreads)
crc_fold_kernel(const uint32_t* __restrict__ first, const uint32_t* __restrict__ count,
                const uint64_t* __restrict__ crc, const uint64_t* __restrict__ len,
                uint64_t* __restrict__ out) {
    __shared__ NibbleTable G[kFoldLevels];  // A_(65536 * 2^L) = x^(2^(19 + L))
    __shared__ uint64_t lens[kFoldThreads / 32];
    __shared__ uint64_t wv[kFoldThreads / 32];
    __shared__ uint64_t xs[2];
    const int tid = threadIdx.x;
    const uint32_t f = first[blockIdx.x];
    const uint32_t n = count[blockIdx.x];
    if (n == 0) {
        if (tid == 0) out[blockIdx.x] = 0ull;  // CRC of the empty string
        return;
    }
    const uint32_t m = n - 1;  // full blocks; block n-1 is the last (maybe short)
    // H = XOR_e G^e v'_e over the full blocks, e = m-1-j counted from the end
    // (v'_e = crc[f + m-1-e], G = A_65536). Thread t owns e in [t per, (t+1) per),
    // per a power of two, by Horner; then a tree over threads whose level-L
    // multiplier is G^(per 2^L) = x^(2^(19 + lp + L)): fixed tables again.
    int lp = 0;
    while ((uint64_t(kFoldThreads) << lp) < m) ++lp;
    const uint32_t per = 1u << lp;
    const int ntab = lp + 10;  // G^(2^i), i < lp + 10 (table i = x^(2^(19+i)))
    {
        const uint4* src = reinterpret_cast<const uint4*>(&g_tables[19 - kFirstPow]);
        uint4* dst = reinterpret_cast<uint4*>(&G[0]);
        for (int i = tid; i < int(sizeof(NibbleTable)) * ntab / 16; i += kFoldThreads) dst[i] = src[i];
    }
    uint64_t mine = 0;  // segment length
    for (uint32_t j = tid; j < n; j += kFoldThreads) mine += len[f + j];
#pragma unroll
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xFFFFFFFFu, mine, o);
    if ((tid & 31) == 0) lens[tid >> 5] = mine;
    __syncthreads();  // lens, tables
    uint64_t total = 0;
#pragma unroll
    for (int w = 0; w < kFoldThreads / 32; ++w) total += lens[w];
    const uint64_t last_len = len[f + m];
    if (tid < 64) {  // warps 0 and 1: the two generic powers, in parallel
        const uint64_t x = x8n_warp(tid < 32 ? last_len : total);
        if ((tid & 31) == 0) xs[tid >> 5] = x;
    }
    const uint64_t* v = crc + f;
    uint64_t acc = 0;
    for (uint32_t d = per; d-- > 0;) {
        const uint64_t e = uint64_t(tid) * per + d;
        acc = mulc(G[0], acc) ^ (e < m ? v[m - 1 - e] : 0ull);
    }
    const int lane = tid & 31, warp = tid >> 5;
    // thread t + 2^L sits 2^L * per blocks EARLIER: it takes the multiplier
    for (int L = 0; L < 5; ++L) {
        const uint64_t other = __shfl_down_sync(0xFFFFFFFFu, acc, 1 << L);
        if ((lane & ((2 << L) - 1)) == 0) acc ^= mulc(G[lp + L], other);
    }
    if (lane == 0) wv[warp] = acc;
    __syncthreads();
    if (warp == 0) {
        acc = wv[lane];
        for (int L = 0; L < 5; ++L) {
            const uint64_t other = __shfl_down_sync(0xFFFFFFFFu, acc, 1 << L);
            if ((lane & ((2 << L) - 1)) == 0) acc ^= mulc(G[lp + 5 + L], other);
        }
    }
    __syncthreads();  // xs (warps 0-1), also when there is no tree level
    if (tid == 0) {
        const uint64_t F = mulmod(acc, xs[0]) ^ v[m];     // full blocks advanced past the last
        out[blockIdx.x] = ~(F ^ mulmod(~0ull, xs[1]));    // 0 for the empty string
    }
}

// persistent grid: SMs x resident CTAs, never more CTAs than blocks
int blocks_grid(uint32_t n_blocks) {
    static int per_device[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int& g = per_device[dev & 63];
    if (g == 0) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, crc_blocks_kernel, kThreads, 0);
        g = std::max(1, sms * std::max(1, per_sm));
    }
    return static_cast<int>(std::min<uint32_t>(n_blocks, static_cast<uint32_t>(g)));
}

}  // namespace

namespace {
uint64_t host_mulmod(uint64_t a, uint64_t b) {
    uint64_t p = 0;
    for (uint64_t m = 1ull << 63; m; m >>= 1) {
        if (a & m) p ^= b;
        b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
}
}  // namespace

extern "C" cudaError_t fdy_crc64_set_constants(const uint64_t* x2k64) {
    cudaError_t e = cudaMemcpyToSymbol(c_x2k, x2k64, sizeof(uint64_t) * 64);
    if (e != cudaSuccess) return e;
    // table of multiplication by K: entry 16 j + v = (v << 4j) * K (linear in
    // the operand, so a lookup per nibble and an XOR give v * K)
    static NibbleTable tables[kNumTables];
    static const bool built = [&] {
        auto fill = [](NibbleTable& t, uint64_t K) {
            for (int j = 0; j < 16; ++j)
                for (int v = 0; v < 16; ++v) t[j][v] = host_mulmod(uint64_t(v) << (4 * j), K);
        };
        for (int k = kFirstPow; k < kFirstPow + kNumTables; ++k) fill(tables[k - kFirstPow], x2k64[k]);
        return true;
    }();
    (void)built;
    return cudaMemcpyToSymbol(g_tables, tables, sizeof tables);
}

extern "C" cudaError_t fdy_launch_crc64_blocks(const unsigned char* base, const FdyCrcBlock* blocks,
                                               uint32_t n_blocks, uint64_t* block_crc,
                                               uint64_t* block_len, cudaStream_t stream) {
    if (n_blocks)
        crc_blocks_kernel<<<blocks_grid(n_blocks), kThreads, 0, stream>>>(base, blocks, n_blocks, block_crc,
                                                                          block_len);
    return cudaGetLastError();
}

extern "C" cudaError_t fdy_launch_crc64_fold(const uint32_t* seg_first_block, const uint32_t* seg_n_blocks,
                                             uint32_t n_segments, uint64_t* block_crc, uint64_t* block_len,
                                             uint64_t* out, cudaStream_t stream) {
    if (n_segments)
        crc_fold_kernel<<<n_segments, kFoldThreads, 0, stream>>>(seg_first_block, seg_n_blocks, block_crc,
                                                                 block_len, out);
    return cudaGetLastError();
}

extern "C" cudaError_t fdy_launch_crc64(const unsigned char* base, const FdyCrcBlock* blocks,
                                        uint32_t n_blocks, const uint32_t* seg_first_block,
                                        const uint32_t* seg_n_blocks, uint32_t n_segments,
                                        uint64_t* scratch_crc, uint64_t* scratch_len,
                                        uint64_t* out, cudaStream_t stream) {
    if (n_segments == 0) return cudaSuccess;
    if (n_blocks)
        crc_blocks_kernel<<<blocks_grid(n_blocks), kThreads, 0, stream>>>(base, blocks, n_blocks, scratch_crc,
                                                                          scratch_len);
    crc_fold_kernel<<<n_segments, kFoldThreads, 0, stream>>>(seg_first_block, seg_n_blocks, scratch_crc,
                                                             scratch_len, out);
    return cudaGetLastError();
}
