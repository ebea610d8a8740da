#!/bin/bash
# Profile the fused materialize kernel on the headline config (qwen3-235b-a22b~).
set -e
cd "$(dirname "$0")/.."
T=paper_2604_06664_b200/fdy_tool
W=/tmp/fdy_prof; rm -rf $W; mkdir -p $W gpurun_out
$T save paper_2604_06664_b200/workloads/qwen3-235b-a22b.spec $W/a plain > /dev/null
$T pack $W/a > /dev/null
NB=$(python3 -c "import json;m=json.load(open('$W/a/manifest'));print('%x'%(m['allocator']['base']+0x10000000000))")
$T gpu-materialize $W/a 3 8 $NB $W/out.fndg 30 | tee gpurun_out/prof_timing.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $T gpu-materialize $W/a 3 8 $NB $W/out2.fndg 3 > /dev/null
ncu --set full --clock-control none --import-source on -k regex:materialize -s 1 -c 1 \
    -o gpurun_out/prof_materialize -f $T gpu-materialize $W/a 3 8 $NB $W/out3.fndg 3 > /dev/null
ncu --set full --clock-control none --import-source on -k regex:crc_blocks -c 1 \
    -o gpurun_out/prof_crc -f $T gpu-crc $W/a/graphs.bin > /dev/null
echo PROFILE-DONE
