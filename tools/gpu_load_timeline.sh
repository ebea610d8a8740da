#!/bin/bash
# Warm-process LOAD timelines on the headline archive (fdy_tool loadbench):
# share_execs and per-template, FOUNDRY_DEBUG phase stamps and driver-call
# accounting; restore lanes 4 / 8. Output: gpurun_out/load_timeline.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=paper_2604_06664_b200/fdy_tool
A=/tmp/driver_study/q
[ -f $A/manifest ] || { rm -rf /tmp/driver_study; mkdir -p /tmp/driver_study; $T save paper_2604_06664_b200/workloads/qwen3-235b-a22b.spec $A > /dev/null; }
{ for rl in 8 4 2; do for mode in share ""; do echo "== loadbench $mode restore lanes $rl"; FOUNDRY_RESTORE_LANES=$rl FOUNDRY_DEBUG=1 timeout 600 $T loadbench $A 0 8 4 $mode 16 2>&1 | grep -E "rep|driver calls|opened|restore done|integrity done"; done; done; } > gpurun_out/load_timeline.txt 2>&1
