#!/bin/bash
# ncu evidence for the bench command (1 GPU): launch list + full sets of the two
# kernels on the LOAD path. Results land in gpurun_out/; summaries go to profiles/.
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 1 --e2e-steps 1 --skip-load --no-cpu-baseline"
$B > /dev/null 2>&1   # writes the archive once (not under the profiler)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_bench.csv $B > gpurun_out/launches_bench.stdout 2>&1
ncu --set full --clock-control none --import-source on -k regex:fdy_materialize -s 2 -c 1 \
    -o gpurun_out/prof_materialize -f $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:crc_blocks -s 1 -c 1 \
    -o gpurun_out/prof_crc -f $B > /dev/null 2>&1
echo PROFILE-DONE
