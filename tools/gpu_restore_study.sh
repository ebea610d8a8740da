#!/bin/bash
# Per-call driver costs of restore + function preparation from T threads
# (fdy_tool restorebench). Output: gpurun_out/restore_study.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=paper_2604_06664_b200/fdy_tool
A=/tmp/driver_study/q
[ -f $A/manifest ] || { rm -rf /tmp/driver_study; mkdir -p /tmp/driver_study; $T save paper_2604_06664_b200/workloads/qwen3-235b-a22b.spec $A > /dev/null; }
timeout 600 $T restorebench $A > gpurun_out/restore_study.txt 2>&1
