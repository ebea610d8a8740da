#!/bin/bash
# ncu --set full of the member pass on the tier-S arena (bench tier_s loop).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline"
$B > /dev/null 2>&1
# launches of fdy_materialize_kernel: 3 warm-up + 3 value + 3 split on the headline, then
# the tier-S loop (3 warm-up, then alternating whole / split): skip into the tier-S ones
ncu --set full --clock-control none --import-source on -k regex:fdy_materialize_kernel -s 13 -c 1 \
    -o gpurun_out/prof_tier_s -f $B > /dev/null 2>&1
echo done
