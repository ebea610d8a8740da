#!/bin/bash
# Driver-cost study on the headline archive (qwen3-235b-a22b~, 512 graphs,
# 12 templates, 9028 distinct kernel functions in 96 libraries):
# library loads, function loads from T threads, instantiate variants, and the
# LOAD phase timeline (FOUNDRY_DEBUG) per mode. Output: gpurun_out/driver_study.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/driver_study.txt
T=paper_2604_06664_b200/fdy_tool
A=/tmp/driver_study/q
rm -rf /tmp/driver_study; mkdir -p /tmp/driver_study
$T save paper_2604_06664_b200/workloads/qwen3-235b-a22b.spec $A > /dev/null
{
echo "== restorebench"; timeout 600 $T restorebench $A
echo "== instbench"; timeout 600 $T instbench $A
for mode in "" "share"; do for i in 1 2 3; do
  echo "== load $mode #$i"
  FOUNDRY_DEBUG=1 timeout 300 $T load $A 0 8 0 $mode 2>&1 | grep -v "^{"
done; done
} > $O 2>&1
