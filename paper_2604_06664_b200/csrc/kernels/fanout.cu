// Pipelined chain fan-out of the template store across GPUs (SURVEY §8(e)
// option ii): GPU r copies chunk k from GPU r-1 as soon as GPU r-1 has it, so
// the store crosses every link once and the chain costs about one store copy
// plus one chunk per hop, instead of GPU0's egress carrying N-1 copies.
//
// Chunk k's arrival is published as a progress word in the receiving GPU's
// own memory (written after the copy in stream order, with release semantics
// at system scope); the next GPU's stream waits on it with a one-thread
// polling kernel (acquire loads through the CUDA IPC / peer mapping) before
// its copy engine pulls the chunk over NVLink. No host round trip per chunk.
#include <cstdint>

#include "fdy_kernels.h"

namespace {

// A link whose wait gave up (failed set) publishes nothing more, so the links
// after it give up too instead of forwarding what it never received.
__global__ void chain_publish_kernel(uint32_t* progress, uint32_t value, const uint32_t* failed) {
    if (failed && *reinterpret_cast<const volatile uint32_t*>(failed)) return;
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(progress), "r"(value) : "memory");
}

// Gives up after timeout_ns (a predecessor that died must not hang this GPU's
// stream): it then sets *failed, and the link's finish reports it.
__global__ void chain_wait_kernel(const uint32_t* progress, uint32_t value, uint64_t timeout_ns,
                                  uint32_t* failed) {
    if (*reinterpret_cast<volatile uint32_t*>(failed)) return;  // an earlier chunk already gave up
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    uint32_t v = 0;
    for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(progress) : "memory");
        if (v >= value) break;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) {
            atomicExch(failed, 1u);
            break;
        }
        __nanosleep(256);
    }
}

}  // namespace

extern "C" cudaError_t fdy_launch_chain_publish(uint32_t* progress, uint32_t value, const uint32_t* failed,
                                                cudaStream_t stream) {
    chain_publish_kernel<<<1, 1, 0, stream>>>(progress, value, failed);
    return cudaGetLastError();
}

extern "C" cudaError_t fdy_launch_chain_wait(const uint32_t* progress, uint32_t value, uint64_t timeout_ns,
                                             uint32_t* failed, cudaStream_t stream) {
    chain_wait_kernel<<<1, 1, 0, stream>>>(progress, value, timeout_ns, failed);
    return cudaGetLastError();
}
