#!/bin/bash
# Floors + ncu of the materialize launch (both grids) on the headline archive.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > gpurun_out/floor_bench.json 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/write_ceiling tools/write_ceiling.cu && /tmp/write_ceiling > gpurun_out/write_ceiling.jsonl
python tools/gpu_floor.py > gpurun_out/gpu_floor.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fdy_(materialize|relocate)" -s 4 -c 2 \
    -o gpurun_out/prof_mat -f python tools/gpu_floor.py > /dev/null 2>&1
echo done
