// GPU-side SAVE: a CUDA graph produced by stream capture ->
// the reference's portable CapturedGraph (graph_model.hpp:115-125), ready for
// serialize_graphs / encode_graph_record.
//
// The reference records graphs inside its simulated driver's stream capture
// (sim_driver.cpp:222-290: per captured op a node with its kernel ref, dims,
// shared memory, function attributes and FLAT argument bytes; edges from the
// op's dependencies). On the GPU the same facts live in the driver's graph:
//   nodes        cuGraphGetNodes (or the capture order the caller recorded)
//   kernel       cuGraphKernelNodeGetParams: CUfunction / CUkernel -> the
//                restored catalog entry (binary hash, name, FuncAttrs)
//   arguments    kernelParams flattened with cuFuncGetParamInfo (offset and
//                size of every parameter), or the `extra` buffer verbatim
//   attributes   cuGraphKernelNodeGetAttribute (cluster dims, scheduling
//                policy, memory-sync domain map). The driver reports its
//                effective value for an attribute nobody set, so an unset
//                attribute reads back as the driver default; and reference
//                cluster dims that do not divide the grid never reach the
//                hardware (the template build skips them).
//   memcpy/set   CUDA_MEMCPY3D / CUDA_MEMSET_NODE_PARAMS -> src, dst, length
//                / dst, value, length
//   edges        cuGraphGetEdges, mapped to node ids
#pragma once

#include <span>

#include <cuda.h>

#include "foundry/gpu_context.hpp"
#include "foundry/graph_model.hpp"

namespace foundry {

// Extracts `graph` (nodes in `order` if given, else cuGraphGetNodes order).
// Raises unresolved_kernel for a kernel that is not a restored catalog entry,
// invalid_argument for node types the portable model has no form for.
CapturedGraph extract_graph(const GpuContext& ctx, CUgraph graph, uint32_t label,
                            std::span<const CUgraphNode> order = {});

}  // namespace foundry
