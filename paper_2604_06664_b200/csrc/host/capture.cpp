// GPU-side SAVE: CUDA graph -> CapturedGraph (see foundry/capture.hpp).
#include "foundry/capture.hpp"

#include <algorithm>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "foundry/driver_api.hpp"
#include "foundry/errors.hpp"

namespace foundry {

namespace {

// The argument bytes of a kernel node, as one flat buffer (the reference's
// KernelNodeParams.arg_buffer, graph_model.hpp:52-61).
std::vector<uint8_t> flatten_arguments(const DriverApi& api, CUfunction fn, const CUDA_KERNEL_NODE_PARAMS& p,
                                       uint32_t node) {
    std::vector<uint8_t> out;
    if (p.extra) {  // launched with CU_LAUNCH_PARAM_BUFFER_POINTER / _SIZE
        const void* buf = nullptr;
        size_t size = 0;
        for (void** e = p.extra; *e != CU_LAUNCH_PARAM_END; e += 2) {
            if (*e == CU_LAUNCH_PARAM_BUFFER_POINTER) buf = e[1];
            else if (*e == CU_LAUNCH_PARAM_BUFFER_SIZE) size = *static_cast<const size_t*>(e[1]);
        }
        require(buf != nullptr || size == 0, Errc::invalid_argument,
                "node " + std::to_string(node) + ": extra launch options without a parameter buffer");
        out.assign(static_cast<const uint8_t*>(buf), static_cast<const uint8_t*>(buf) + size);
        return out;
    }
    if (!p.kernelParams) return out;  // a kernel without parameters
    require(api.cuFuncGetParamInfo != nullptr, Errc::device_unavailable,
            "cuFuncGetParamInfo (CUDA 12.4+) is needed to flatten captured kernel parameters");
    for (size_t i = 0;; ++i) {
        size_t off = 0, size = 0;
        if (api.cuFuncGetParamInfo(fn, i, &off, &size) != CUDA_SUCCESS) break;  // past the last
        if (out.size() < off + size) out.resize(off + size, 0);
        std::memcpy(out.data() + off, p.kernelParams[i], size);
    }
    return out;
}

KernelNodeAttrs node_attributes(const DriverApi& api, CUgraphNode n) {
    KernelNodeAttrs a;
    CUkernelNodeAttrValue v{};
    if (api.cuGraphKernelNodeGetAttribute(n, CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION, &v) == CUDA_SUCCESS &&
        v.clusterDim.x * v.clusterDim.y * v.clusterDim.z > 1)
        a.cluster_dim = Dim3{v.clusterDim.x, v.clusterDim.y, v.clusterDim.z};
    v = {};
    if (api.cuGraphKernelNodeGetAttribute(n, CU_LAUNCH_ATTRIBUTE_CLUSTER_SCHEDULING_POLICY_PREFERENCE, &v) ==
        CUDA_SUCCESS)
        a.cluster_scheduling_policy_preference = static_cast<int32_t>(v.clusterSchedulingPolicyPreference);
    v = {};
    if (api.cuGraphKernelNodeGetAttribute(n, CU_LAUNCH_ATTRIBUTE_MEM_SYNC_DOMAIN_MAP, &v) == CUDA_SUCCESS) {
        a.mem_sync_domain_map_default = v.memSyncDomainMap.default_;
        a.mem_sync_domain_map_remote = v.memSyncDomainMap.remote;
    }
    return a;
}

}  // namespace

CapturedGraph extract_graph(const GpuContext& ctx, CUgraph graph, uint32_t label,
                            std::span<const CUgraphNode> order) {
    const DriverApi& api = driver();
    std::vector<CUgraphNode> nodes(order.begin(), order.end());
    if (nodes.empty()) {
        size_t n = 0;
        cu_check(api.cuGraphGetNodes(graph, nullptr, &n), "cuGraphGetNodes(count)");
        nodes.resize(n);
        if (n) cu_check(api.cuGraphGetNodes(graph, nodes.data(), &n), "cuGraphGetNodes");
    }
    std::unordered_map<CUgraphNode, uint32_t> id;
    for (uint32_t i = 0; i < nodes.size(); ++i) id.emplace(nodes[i], i);

    CapturedGraph g;
    g.label = label;
    g.nodes.resize(nodes.size());
    for (uint32_t i = 0; i < nodes.size(); ++i) {
        GraphNode& out = g.nodes[i];
        out.id = i;
        CUgraphNodeType t;
        cu_check(api.cuGraphNodeGetType(nodes[i], &t), "cuGraphNodeGetType");
        switch (t) {
            case CU_GRAPH_NODE_TYPE_KERNEL: {
                CUDA_KERNEL_NODE_PARAMS p;
                std::memset(&p, 0, sizeof p);
                cu_check(api.cuGraphKernelNodeGetParams(nodes[i], &p), "cuGraphKernelNodeGetParams");
                const GpuContext::Kernel* K = ctx.kernel_by_handle(p.func, p.kern);
                require(K != nullptr, Errc::unresolved_kernel,
                        "node " + std::to_string(i) + " launches a function that is not a restored catalog entry");
                KernelNodeParams kp;
                kp.grid = Dim3{p.gridDimX, p.gridDimY, p.gridDimZ};
                kp.block = Dim3{p.blockDimX, p.blockDimY, p.blockDimZ};
                kp.shared_mem_bytes = p.sharedMemBytes;
                kp.kernel = KernelRef{K->binary_hash, K->name};
                kp.func_attrs = K->attrs;
                kp.arg_buffer = flatten_arguments(api, p.func ? p.func : ctx.function(*K), p, i);
                out.type = NodeType::Kernel;
                out.attrs = node_attributes(api, nodes[i]);
                out.params = std::move(kp);
                break;
            }
            case CU_GRAPH_NODE_TYPE_MEMCPY: {
                CUDA_MEMCPY3D c;
                std::memset(&c, 0, sizeof c);
                cu_check(api.cuGraphMemcpyNodeGetParams(nodes[i], &c), "cuGraphMemcpyNodeGetParams");
                require(c.Height <= 1 && c.Depth <= 1, Errc::invalid_argument,
                        "node " + std::to_string(i) + ": only 1-D copies have a portable form");
                out.type = NodeType::Memcpy;
                out.params = MemcpyParams{c.srcDevice + c.srcXInBytes, c.dstDevice + c.dstXInBytes, c.WidthInBytes};
                break;
            }
            case CU_GRAPH_NODE_TYPE_MEMSET: {
                CUDA_MEMSET_NODE_PARAMS m;
                std::memset(&m, 0, sizeof m);
                cu_check(api.cuGraphMemsetNodeGetParams(nodes[i], &m), "cuGraphMemsetNodeGetParams");
                require(m.height <= 1, Errc::invalid_argument,
                        "node " + std::to_string(i) + ": only 1-D memsets have a portable form");
                out.type = NodeType::Memset;
                out.params = MemsetParams{m.dst, m.value, uint64_t(m.width) * m.elementSize};
                break;
            }
            case CU_GRAPH_NODE_TYPE_EMPTY:
                out.type = NodeType::Empty;
                out.params = EmptyParams{};
                break;
            default:
                raise(Errc::invalid_argument,
                      "node " + std::to_string(i) + ": node type " + std::to_string(int(t)) +
                          " has no form in the portable graph model");
        }
    }
    size_t ne = 0;
    cu_check(api.cuGraphGetEdges(graph, nullptr, nullptr, &ne), "cuGraphGetEdges(count)");
    std::vector<CUgraphNode> from(ne), to(ne);
    if (ne) cu_check(api.cuGraphGetEdges(graph, from.data(), to.data(), &ne), "cuGraphGetEdges");
    for (size_t e = 0; e < ne; ++e) {
        const auto a = id.find(from[e]), b = id.find(to[e]);
        require(a != id.end() && b != id.end(), Errc::invalid_argument, "edge references a node outside the order");
        g.edges.push_back(GraphEdge{a->second, b->second});
    }
    g.canonicalize();
    return g;
}

}  // namespace foundry
