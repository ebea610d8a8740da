// GPU CRC-64/XZ for archive integrity: replaces the
// reference's single-threaded byte-at-a-time walk over every archive file
// (verify_archive_integrity, pipeline.cpp:411-417; Crc64::update, hash.cpp:53-61)
// with an HBM-resident, chunk-parallel computation.
//
// Algebra: for the standard CRC-64/XZ (init = xorout = ~0, reflected),
//     crc(A || B) = mulmod(x^(8|B|), crc(A)) ^ crc(B)
// with polynomial products taken mod P in the reflected bit order. Each thread
// CRCs 256 contiguous bytes with slicing-by-8 tables held in shared memory;
// a CTA folds its 256 partial CRCs (64 KiB block) with a tree of such
// combines; a second kernel folds the blocks of each segment the same way.
#include <cstdint>

#include "fdy_kernels.h"

namespace {

constexpr uint64_t kPoly = 0xC96C5795D7870F42ull;
constexpr int kThreads = 256;
constexpr uint32_t kBytesPerThread = kCrcBlockBytes / kThreads;
static_assert(kBytesPerThread % 16 == 0, "thread span must be a multiple of 16 bytes");

__constant__ uint64_t c_x2k[64];  // x^(2^k) mod P, k = 0..63 (host-computed)

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

__device__ __forceinline__ uint64_t combine(uint64_t crc_a, uint64_t crc_b, uint64_t len_b) {
    return len_b ? (mulmod(x8n(len_b), crc_a) ^ crc_b) : crc_a;
}

__global__ void __launch_bounds__(kThreads)
crc_blocks_kernel(const unsigned char* __restrict__ base, const FdyCrcBlock* __restrict__ blocks,
                  uint64_t* __restrict__ out_crc, uint64_t* __restrict__ out_len) {
    __shared__ uint64_t T[8][256];
    __shared__ uint64_t part[kThreads];
    __shared__ uint64_t plen[kThreads];
    const int tid = threadIdx.x;

    {  // slicing-by-8 tables
        uint64_t c = static_cast<uint64_t>(tid);
#pragma unroll
        for (int b = 0; b < 8; ++b) c = (c & 1ull) ? (c >> 1) ^ kPoly : c >> 1;
        T[0][tid] = c;
        __syncthreads();
#pragma unroll
        for (int k = 1; k < 8; ++k) {
            const uint64_t prev = T[k - 1][tid];
            T[k][tid] = (prev >> 8) ^ T[0][prev & 0xFF];
            __syncthreads();
        }
    }

    const FdyCrcBlock blk = blocks[blockIdx.x];
    const uint32_t lo = umin(blk.length, tid * kBytesPerThread);
    const uint32_t hi = umin(blk.length, lo + kBytesPerThread);
    const unsigned char* p = base + blk.offset + lo;
    uint64_t c = ~0ull;
    uint32_t i = 0;
    const uint32_t n = hi - lo;
    for (; i + 16 <= n; i += 16) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p + i));
        uint64_t w = (uint64_t(v.y) << 32) | v.x;
        c ^= w;
        c = T[7][c & 0xFF] ^ T[6][(c >> 8) & 0xFF] ^ T[5][(c >> 16) & 0xFF] ^
            T[4][(c >> 24) & 0xFF] ^ T[3][(c >> 32) & 0xFF] ^ T[2][(c >> 40) & 0xFF] ^
            T[1][(c >> 48) & 0xFF] ^ T[0][c >> 56];
        w = (uint64_t(v.w) << 32) | v.z;
        c ^= w;
        c = T[7][c & 0xFF] ^ T[6][(c >> 8) & 0xFF] ^ T[5][(c >> 16) & 0xFF] ^
            T[4][(c >> 24) & 0xFF] ^ T[3][(c >> 32) & 0xFF] ^ T[2][(c >> 40) & 0xFF] ^
            T[1][(c >> 48) & 0xFF] ^ T[0][c >> 56];
    }
    for (; i < n; ++i) c = (c >> 8) ^ T[0][(c ^ p[i]) & 0xFF];
    part[tid] = n ? ~c : 0ull;  // CRC of the empty string is 0
    plen[tid] = n;
    __syncthreads();

    // fold: crc(run_i || run_{i+s}) with |run_{i+s}| = plen
    for (int s = 1; s < kThreads; s <<= 1) {
        if ((tid & (2 * s - 1)) == 0 && tid + s < kThreads) {
            part[tid] = combine(part[tid], part[tid + s], plen[tid + s]);
            plen[tid] += plen[tid + s];
        }
        __syncthreads();
    }
    if (tid == 0) {
        out_crc[blockIdx.x] = part[0];
        out_len[blockIdx.x] = plen[0];
    }
}

__global__ void __launch_bounds__(1024)
crc_fold_kernel(const uint32_t* __restrict__ first, const uint32_t* __restrict__ count,
                uint64_t* __restrict__ crc, uint64_t* __restrict__ len, uint64_t* __restrict__ out) {
    const uint32_t f = first[blockIdx.x];
    const uint32_t n = count[blockIdx.x];
    for (uint32_t s = 1; s < n; s <<= 1) {
        for (uint32_t i = threadIdx.x * 2 * s; i + s < n; i += blockDim.x * 2 * s) {
            crc[f + i] = combine(crc[f + i], crc[f + i + s], len[f + i + s]);
            len[f + i] += len[f + i + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = n ? crc[f] : 0ull;
}

}  // namespace

extern "C" cudaError_t fdy_crc64_set_constants(const uint64_t* x2k64) {
    return cudaMemcpyToSymbol(c_x2k, x2k64, sizeof(uint64_t) * 64);
}

extern "C" cudaError_t fdy_launch_crc64_blocks(const unsigned char* base, const FdyCrcBlock* blocks,
                                               uint32_t n_blocks, uint64_t* block_crc,
                                               uint64_t* block_len, cudaStream_t stream) {
    if (n_blocks) crc_blocks_kernel<<<n_blocks, kThreads, 0, stream>>>(base, blocks, block_crc, block_len);
    return cudaGetLastError();
}

extern "C" cudaError_t fdy_launch_crc64_fold(const uint32_t* seg_first_block, const uint32_t* seg_n_blocks,
                                             uint32_t n_segments, uint64_t* block_crc, uint64_t* block_len,
                                             uint64_t* out, cudaStream_t stream) {
    if (n_segments)
        crc_fold_kernel<<<n_segments, 1024, 0, stream>>>(seg_first_block, seg_n_blocks, block_crc, block_len,
                                                         out);
    return cudaGetLastError();
}

extern "C" cudaError_t fdy_launch_crc64(const unsigned char* base, const FdyCrcBlock* blocks,
                                        uint32_t n_blocks, const uint32_t* seg_first_block,
                                        const uint32_t* seg_n_blocks, uint32_t n_segments,
                                        uint64_t* scratch_crc, uint64_t* scratch_len,
                                        uint64_t* out, cudaStream_t stream) {
    if (n_segments == 0) return cudaSuccess;
    if (n_blocks) crc_blocks_kernel<<<n_blocks, kThreads, 0, stream>>>(base, blocks, scratch_crc, scratch_len);
    crc_fold_kernel<<<n_segments, 1024, 0, stream>>>(seg_first_block, seg_n_blocks, scratch_crc,
                                                     scratch_len, out);
    return cudaGetLastError();
}
