#!/bin/bash
# Driver-cost study of the full LOAD on the headline archive: per-group build /
# instantiate under module-loading, edge-shape and builder-lane variants.
cd "$(dirname "$0")/.."
T=paper_2604_06664_b200/fdy_tool
W=/tmp/fdy_exp; rm -rf $W; mkdir -p $W gpurun_out
$T save paper_2604_06664_b200/workloads/qwen3-235b-a22b.spec $W/a plain > /dev/null
$T pack $W/a > /dev/null
for v in "" "CUDA_MODULE_LOADING=EAGER" "FOUNDRY_BUILD_LANES=4" "CUDA_MODULE_LOADING=EAGER FOUNDRY_BUILD_LANES=4"; do
  echo "=== $v"
  for i in 1 2; do env $v FOUNDRY_DEBUG=1 $T load $W/a 0 8 2>&1 | grep -E "group 0:|group 11:|loaded|restore done|instantiated group" | tail -6; done
done
