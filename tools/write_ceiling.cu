// Write-bandwidth ceiling probe (tools only, not part of the product).
// Streams `bytes` of output from shared memory with cp.async.bulk stores
// (the materialize kernel's store path) and with plain st.global.v4, cold
// L2, CUDA events; prints one JSON line per variant and size.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_ceiling tools/write_ceiling.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kTile = 16384;

__global__ void __launch_bounds__(256) bulk_store_kernel(unsigned char* out, uint64_t n_tiles) {
    extern __shared__ __align__(128) unsigned char buf[];
    for (int i = threadIdx.x; i < kTile / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(buf)[i] = make_uint4(i, 1, 2, 3);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + t * kTile),
                     "r"(s), "r"(kTile) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(256) st_v4_kernel(uint4* out, uint64_t n) {
    const uint4 v = make_uint4(1, 2, 3, 4);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = v;
}

__global__ void __launch_bounds__(256) copy_v4_kernel(uint4* out, const uint4* in, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = __ldg(in + i);
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint64_t max_bytes = 2048ull << 20;
    unsigned char *out, *in, *flush;
    CK(cudaMalloc(&out, max_bytes));
    CK(cudaMalloc(&in, max_bytes));
    CK(cudaMalloc(&flush, 512ull << 20));
    CK(cudaFuncSetAttribute(bulk_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTile));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const uint64_t sizes[] = {147161088ull, 1024ull << 20};
    for (uint64_t bytes : sizes) {
        for (int variant = 0; variant < 4; ++variant) {
            std::vector<float> ms;
            for (int r = 0; r < 12; ++r) {
                CK(cudaMemset(flush, r, 512ull << 20));
                CK(cudaDeviceSynchronize());
                CK(cudaEventRecord(e0));
                if (variant == 0)
                    bulk_store_kernel<<<sms * 8, 256, kTile>>>(out, bytes / kTile);
                else if (variant == 1)
                    bulk_store_kernel<<<sms * 2, 256, kTile>>>(out, bytes / kTile);
                else if (variant == 2)
                    st_v4_kernel<<<sms * 8, 256>>>(reinterpret_cast<uint4*>(out), bytes / 16);
                else
                    copy_v4_kernel<<<sms * 8, 256>>>(reinterpret_cast<uint4*>(out),
                                                     reinterpret_cast<const uint4*>(in), bytes / 16);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float t;
                CK(cudaEventElapsedTime(&t, e0, e1));
                if (r >= 2) ms.push_back(t);
            }
            std::sort(ms.begin(), ms.end());
            const char* names[] = {"bulk_store grid=8xSM", "bulk_store grid=2xSM", "st.global.v4 grid=8xSM",
                                   "copy ld/st.v4 grid=8xSM"};
            const double moved = variant == 3 ? 2.0 * bytes : double(bytes);
            printf("{\"variant\": \"%s\", \"bytes\": %llu, \"best_us\": %.2f, \"median_us\": %.2f, "
                   "\"GBps_median\": %.1f}\n",
                   names[variant], (unsigned long long)bytes, ms.front() * 1e3, ms[ms.size() / 2] * 1e3,
                   moved / (ms[ms.size() / 2] * 1e-3) / 1e9);
        }
    }
    return 0;
}
