#!/bin/bash
# Driver-cost study: library restore / function loading on the headline archive.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
A=/tmp/foundry_bench_qwen3-235b-a22b/b200
T=paper_2604_06664_b200/fdy_tool
python -c "import json;m=json.load(open('$A/manifest'));print('files',len(m['file_digests']))"
ls $A/binaries | wc -l; du -sh $A/binaries
$T restorebench $A
for v in "" "CUDA_MODULE_LOADING=EAGER"; do
  echo "=== $v"
  for i in 1 2; do env $v FOUNDRY_DEBUG=1 $T load $A 0 8 2>&1 | grep -E "loaded|done|group 0:|group 11:" | tail -12; done
done
