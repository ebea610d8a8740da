// Probe (tools only): can a kernel OUTSIDE a graph update the parameters and
// grid of device-updatable kernel nodes of an instantiated graph, and does the
// next host cudaGraphLaunch see the update?  Also times N node updates.
//   nvcc -gencode arch=compute_100a,code=sm_100a -rdc=true -O3 tools/devupdate_probe.cu -lcudadevrt -o /tmp/dup
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Args { unsigned long long v[40]; };  // 320-byte parameter block like a trace kernel

__global__ void body(Args a, unsigned long long* out, int id) {
    if (threadIdx.x == 0) atomicAdd(out + id, a.v[0] + a.v[39] * gridDim.x);
}

__global__ void updater(const cudaGraphDeviceNode_t* nodes, int n, unsigned long long base, unsigned gx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Args a;
    for (int k = 0; k < 40; ++k) a.v[k] = 0;
    a.v[0] = base + i;
    a.v[39] = 1;
    cudaGraphKernelNodeSetParam(nodes[i], 0, &a, sizeof a);
    cudaGraphKernelNodeSetGridDim(nodes[i], dim3(gx, 1, 1));
}

int main() {
    const int N = 1024;
    unsigned long long* out;
    CK(cudaMalloc(&out, N * 8));
    CK(cudaMemset(out, 0, N * 8));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    std::vector<cudaGraphNode_t> nodes(N);
    Args a0{};
    for (int i = 0; i < N; ++i) {
        int id = i;
        void* params[3] = {&a0, &out, &id};
        cudaKernelNodeParams p{};
        p.func = (void*)body;
        p.gridDim = dim3(1);
        p.blockDim = dim3(32);
        p.kernelParams = params;
        CK(cudaGraphAddKernelNode(&nodes[i], g, i ? &nodes[i - 1] : nullptr, i ? 1 : 0, &p));
        cudaLaunchAttributeValue v{};
        v.deviceUpdatableKernelNode.deviceUpdatable = 1;
        CK(cudaGraphKernelNodeSetAttribute(nodes[i], cudaLaunchAttributeDeviceUpdatableKernelNode, &v));
    }
    std::vector<cudaGraphDeviceNode_t> dn(N);
    for (int i = 0; i < N; ++i) {
        cudaLaunchAttributeValue v{};
        CK(cudaGraphKernelNodeGetAttribute(nodes[i], cudaLaunchAttributeDeviceUpdatableKernelNode, &v));
        dn[i] = v.deviceUpdatableKernelNode.devNode;
    }
    printf("devNode[0]=%p devNode[1]=%p\n", (void*)dn[0], (void*)dn[1]);
    cudaGraphExec_t x;
    CK(cudaGraphInstantiate(&x, g, 0));
    CK(cudaGraphUpload(x, s));
    cudaGraphDeviceNode_t* d_dn;
    CK(cudaMalloc(&d_dn, N * sizeof(cudaGraphDeviceNode_t)));
    // re-query after instantiate (handles may only be valid then)
    for (int i = 0; i < N; ++i) {
        cudaLaunchAttributeValue v{};
        CK(cudaGraphKernelNodeGetAttribute(nodes[i], cudaLaunchAttributeDeviceUpdatableKernelNode, &v));
        if (v.deviceUpdatableKernelNode.devNode != dn[i]) printf("node %d handle changed after instantiate\n", i);
        dn[i] = v.deviceUpdatableKernelNode.devNode;
    }
    CK(cudaMemcpy(d_dn, dn.data(), N * sizeof(cudaGraphDeviceNode_t), cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemsetAsync(out, 0, N * 8, s));
        CK(cudaEventRecord(e0, s));
        updater<<<(N + 127) / 128, 128, 0, s>>>(d_dn, N, 1000ull * (rep + 1), 2 + rep);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1, s));
        CK(cudaGraphLaunch(x, s));
        CK(cudaStreamSynchronize(s));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        std::vector<unsigned long long> h(N);
        CK(cudaMemcpy(h.data(), out, N * 8, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int i = 0; i < N; ++i) {
            const unsigned long long want = (1000ull * (rep + 1) + i + 1 * (2 + rep)) * (2 + rep);
            if (h[i] != want) { if (bad < 3) printf("node %d got %llu want %llu\n", i, h[i], want); ++bad; }
        }
        printf("rep %d: updater %.3f us for %d nodes, mismatches %d\n", rep, ms * 1e3, N, bad);
    }
    return 0;
}
