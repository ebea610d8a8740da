# A/B: CUDA_MODULE_LOADING lazy vs eager for a fresh-process LOAD (fdy_tool load)
cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > gpurun_out/modload_bench.log 2>&1 || tail -5 gpurun_out/modload_bench.log
A=/tmp/foundry_bench_qwen3-235b-a22b/b200
ls $A | head -3
T=paper_2604_06664_b200/fdy_tool
$T load $A 0 8 2>&1 | tail -2
for m in LAZY EAGER LAZY EAGER; do
  echo "== $m"
  s=$(date +%s.%N)
  CUDA_MODULE_LOADING=$m $T load $A 0 8 2>&1 | grep -E "loaded" | tail -2
  e=$(date +%s.%N); echo "wall $(echo "$e - $s" | bc) s"
done
