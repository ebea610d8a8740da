#!/bin/bash
# ncu evidence for the bench command (1 GPU): launch list + full sets of the
# kernels on the path. Results land in gpurun_out/; summaries go to profiles/.
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline --skip-tier-s"
$B > /dev/null 2>&1   # writes the archive once (not under the profiler)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_bench.csv $B > gpurun_out/launches_bench.stdout 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fdy_(materialize|relocate)" -s 6 -c 2 \
    -o gpurun_out/prof_materialize -f $B > /dev/null 2>&1
# GPU CRC-64 at archive scale (277 MB in 3 segments)
ncu --set full --clock-control none --import-source on -k regex:crc_ -s 2 -c 2 \
    -o gpurun_out/prof_crc -f python tools/gpu_crc_bench.py > /dev/null 2>&1
python tools/gpu_crc_bench.py > gpurun_out/crc_bench.json
# the device-side serve kernel (LoadOptions.device_updates), one launch
ncu --set full --clock-control none --import-source on -k regex:fdy_serve -s 20 -c 1 \
    -o gpurun_out/prof_serve -f python tools/gpu_serve_bench.py /tmp/foundry_bench_qwen3-235b-a22b/b200 device_updates > /dev/null 2>&1
python tools/gpu_serve_bench.py > gpurun_out/serve_bench.json
python tools/gpu_floor.py > gpurun_out/gpu_floor.json 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/write_ceiling tools/write_ceiling.cu && /tmp/write_ceiling > gpurun_out/write_ceiling.jsonl
echo PROFILE-DONE
