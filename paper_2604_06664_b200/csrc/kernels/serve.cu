// Device-side serve for sm_100a (reference ServingSet::serve -> exec_update,
// templater.cpp:177-188, sim_driver.cpp:365-398): apply member m's parameters
// to its template's instantiated graph from the GPU, reading them straight out
// of the member-image arena the materialize kernel wrote in HBM.
//
// The template's kernel nodes are device-updatable
// (CU_LAUNCH_ATTRIBUTE_DEVICE_UPDATABLE_KERNEL_NODE); one warp per node
// calls cudaGraphKernelNodeSetParam (16-byte slices of the argument block) and
// cudaGraphKernelNodeSetGridDim. A device update cannot change a node's
// function, block dims or dynamic shared memory, and memcpy / memset nodes
// have no device-side update: fdy_serve_plan_kernel records, once per LOAD,
// which members need the host path and every member's memop records, so the
// host applies memops with cuGraphExec*NodeSetParams without a readback and
// serve() never waits on the device. No host copy of the member image is needed.
//
// Compiled with -rdc=true and device-linked against libcudadevrt (the device
// graph-update API lives in the device runtime).
#include <cstdint>

#include "fdy_kernels.h"

namespace {

constexpr int kServeThreads = 128;  // 4 nodes per CTA: one warp per node

// One warp per node: lane l writes argument bytes [16 l, 16 l + 16) with its
// own cudaGraphKernelNodeSetParam (disjoint ranges of the node's parameter
// block), lane 0 the grid; a single thread per node was latency-bound on the
// device runtime's byte copy (20 us for 1036 nodes).
__global__ void __launch_bounds__(kServeThreads)
fdy_serve_kernel(const FdyServeArgs a) {
    const uint32_t n = blockIdx.x * (kServeThreads / 32) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (n >= a.n_nodes) return;
    const fdt_node d = reinterpret_cast<const fdt_node*>(a.image)[n];
    const FdyServeNode& s = a.nodes[n];
    const unsigned char* blob = a.image + 48ull * a.n_nodes + d.blob_off;
    uint8_t flag = 0;
    if (d.type == 0 && s.devnode != nullptr && d.kernel == s.kernel && d.block[0] == s.block[0] &&
        d.block[1] == s.block[1] && d.block[2] == s.block[2] && d.shmem == s.shmem) {
        const cudaGraphDeviceNode_t node = reinterpret_cast<cudaGraphDeviceNode_t>(s.devnode);
        bool ok = true;
        for (uint32_t off = 16 * lane; off < s.param_bytes; off += 16 * 32)
            ok &= cudaGraphKernelNodeSetParam(node, off, blob + off, min(16u, s.param_bytes - off)) == cudaSuccess;
        if (lane == 0) ok &= cudaGraphKernelNodeSetGridDim(node, dim3(d.grid[0], d.grid[1], d.grid[2])) == cudaSuccess;
        if (a.inject_failure) ok = false;
        if (!__all_sync(0xFFFFFFFFu, ok)) {
            flag = 2;  // the host re-applies the whole member
            // nothing waits for this kernel: the word is checked at the next
            // synchronization point (replay), which re-applies on the host
            if (lane == 0 && a.error_word) {
                a.member_failed[a.member] = 1;
                __threadfence_system();
                atomicOr(a.error_word, 1u);
            }
        }
    } else if (d.type == 1 || d.type == 2) {
        flag = 1;  // memop: host SetParams from the record below
        if (lane < 3 && a.host_records) a.host_records[3ull * n + lane] = reinterpret_cast<const uint64_t*>(blob)[lane];
    } else if (d.type == 0) {
        flag = 2;  // function / block / shmem changed: host path
    }
    if (lane == 0 && a.host_flags) a.host_flags[n] = flag;
}

// One CTA per member: device-applicability flag and memop records (see FdyServePlanArgs).
__global__ void __launch_bounds__(kServeThreads)
fdy_serve_plan_kernel(const FdyServePlanArgs a) {
    __shared__ int needs_host;
    const uint32_t m = blockIdx.x;
    if (threadIdx.x == 0) needs_host = 0;
    __syncthreads();
    const uint32_t g = a.member_group[m];
    const FdyServeNode* nodes = a.group_nodes[g];
    const uint32_t nn = a.group_n_nodes[g];
    const unsigned char* image = a.arena + a.member_off[m];
    for (uint32_t n = threadIdx.x; n < nn; n += kServeThreads) {
        const fdt_node d = reinterpret_cast<const fdt_node*>(image)[n];
        const FdyServeNode& s = nodes[n];
        if (d.type == 0) {
            if (s.devnode == nullptr || d.kernel != s.kernel || d.block[0] != s.block[0] ||
                d.block[1] != s.block[1] || d.block[2] != s.block[2] || d.shmem != s.shmem)
                needs_host = 1;
        } else if ((d.type == 1 || d.type == 2) && s.memop_slot >= 0) {
            const uint64_t* r = reinterpret_cast<const uint64_t*>(image + 48ull * nn + d.blob_off);
            uint64_t* out = a.records + 3ull * (a.memop_base[m] + uint32_t(s.memop_slot));
            out[0] = r[0], out[1] = r[1], out[2] = r[2];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) a.member_host[m] = uint8_t(needs_host);
}

}  // namespace

extern "C" cudaError_t fdy_launch_serve_plan(const FdyServePlanArgs* args, cudaStream_t stream) {
    if (args->n_members == 0) return cudaSuccess;
    fdy_serve_plan_kernel<<<args->n_members, kServeThreads, 0, stream>>>(*args);
    return cudaGetLastError();
}

extern "C" cudaError_t fdy_launch_serve(const FdyServeArgs* args, cudaStream_t stream) {
    if (args->n_nodes == 0) return cudaSuccess;
    const uint32_t per_cta = kServeThreads / 32;
    fdy_serve_kernel<<<(args->n_nodes + per_cta - 1) / per_cta, kServeThreads, 0, stream>>>(*args);
    return cudaGetLastError();
}
