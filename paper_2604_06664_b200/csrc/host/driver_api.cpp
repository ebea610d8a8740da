// Runtime resolution of the CUDA driver entry points (see driver_api.hpp).
#include "foundry/driver_api.hpp"

#include <mutex>
#include <string>

#include <cuda_runtime.h>

#include "foundry/device.hpp"
#include "foundry/errors.hpp"

namespace foundry {

namespace {

DriverApi g_api{};
std::once_flag g_once;
std::string g_error;

template <typename Fn>
void resolve(Fn& slot, const char* symbol, unsigned version = 12000) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    const cudaError_t e = cudaGetDriverEntryPointByVersion(symbol, &p, version, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || p == nullptr) {
        cudaGetLastError();
        if (g_error.empty()) g_error = std::string("cannot resolve driver entry point ") + symbol;
        return;
    }
    slot = reinterpret_cast<Fn>(p);
}

void load_all() {
    if (!cuda_available()) {
        g_error = "no CUDA driver/device visible (the B200 path has no CPU fallback)";
        return;
    }
#define FDY_RESOLVE(name) resolve(g_api.name, #name)
    FDY_RESOLVE(cuCtxGetCurrent);
    FDY_RESOLVE(cuGetErrorName);
    FDY_RESOLVE(cuGetErrorString);
    FDY_RESOLVE(cuMemAddressReserve);
    FDY_RESOLVE(cuMemAddressFree);
    FDY_RESOLVE(cuMemCreate);
    FDY_RESOLVE(cuMemRelease);
    FDY_RESOLVE(cuMemMap);
    FDY_RESOLVE(cuMemUnmap);
    FDY_RESOLVE(cuMemSetAccess);
    FDY_RESOLVE(cuMemGetAllocationGranularity);
    FDY_RESOLVE(cuLibraryLoadData);
    FDY_RESOLVE(cuLibraryUnload);
    FDY_RESOLVE(cuLibraryGetKernel);
    FDY_RESOLVE(cuLibraryGetGlobal);
    FDY_RESOLVE(cuKernelGetFunction);
    FDY_RESOLVE(cuFuncSetAttribute);
    FDY_RESOLVE(cuFuncGetAttribute);
    FDY_RESOLVE(cuKernelSetAttribute);
    FDY_RESOLVE(cuCtxGetDevice);
    FDY_RESOLVE(cuGraphCreate);
    FDY_RESOLVE(cuGraphDestroy);
    FDY_RESOLVE(cuGraphAddKernelNode);
    FDY_RESOLVE(cuGraphAddMemcpyNode);
    FDY_RESOLVE(cuGraphAddMemsetNode);
    FDY_RESOLVE(cuGraphAddEmptyNode);
    FDY_RESOLVE(cuGraphAddDependencies);
    FDY_RESOLVE(cuGraphKernelNodeSetAttribute);
    resolve(g_api.cuGraphInstantiate, "cuGraphInstantiateWithFlags");  // not the legacy _v2 ABI
    FDY_RESOLVE(cuGraphExecDestroy);
    FDY_RESOLVE(cuGraphExecKernelNodeSetParams);
    FDY_RESOLVE(cuGraphExecMemcpyNodeSetParams);
    FDY_RESOLVE(cuGraphExecMemsetNodeSetParams);
    FDY_RESOLVE(cuGraphLaunch);
    FDY_RESOLVE(cuLaunchKernel);
    FDY_RESOLVE(cuMemsetD8Async);
    FDY_RESOLVE(cuMemsetD32Async);
    FDY_RESOLVE(cuGraphGetNodes);
    FDY_RESOLVE(cuGraphGetEdges);
    FDY_RESOLVE(cuGraphNodeGetType);
    FDY_RESOLVE(cuGraphKernelNodeGetParams);
    FDY_RESOLVE(cuGraphMemcpyNodeGetParams);
    FDY_RESOLVE(cuGraphMemsetNodeGetParams);
    FDY_RESOLVE(cuGraphKernelNodeGetAttribute);
    resolve(g_api.cuFuncGetParamInfo, "cuFuncGetParamInfo", 12040);
    FDY_RESOLVE(cuLaunchKernelEx);
    resolve(g_api.cuFuncLoad, "cuFuncLoad", 12040);
    FDY_RESOLVE(cuGraphUpload);
    resolve(g_api.cuLibraryGetKernelCount, "cuLibraryGetKernelCount", 12040);
    resolve(g_api.cuLibraryEnumerateKernels, "cuLibraryEnumerateKernels", 12040);
    resolve(g_api.cuKernelGetName, "cuKernelGetName", 12040);
#undef FDY_RESOLVE
}

}  // namespace

const DriverApi& driver() {
    std::call_once(g_once, load_all);
    require(g_error.empty(), Errc::device_unavailable, g_error);
    return g_api;
}

void cu_check(CUresult r, const char* what) {
    if (r == CUDA_SUCCESS) return;
    const char* name = "CUDA_ERROR";
    const char* text = "";
    if (g_api.cuGetErrorName) g_api.cuGetErrorName(r, &name);
    if (g_api.cuGetErrorString) g_api.cuGetErrorString(r, &text);
    raise(Errc::cuda_error, std::string(what) + " failed: " + name + " (" + text + ")");
}

}  // namespace foundry
