#!/bin/bash
# restorebench under CUDA_MODULE_LOADING=EAGER vs the default (lazy): does
# eager loading make the catalog's function loads cheaper per function?
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=paper_2604_06664_b200/fdy_tool
A=/tmp/driver_study/q
[ -f $A/manifest ] || { rm -rf /tmp/driver_study; mkdir -p /tmp/driver_study; $T save paper_2604_06664_b200/workloads/qwen3-235b-a22b.spec $A > /dev/null; }
{ echo "== LAZY"; timeout 300 $T restorebench $A; echo "== EAGER"; CUDA_MODULE_LOADING=EAGER timeout 300 $T restorebench $A; } > gpurun_out/eager_study.txt 2>&1
