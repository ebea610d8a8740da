# A/B: CUDA_MODULE_LOADING lazy vs eager for a fresh-process LOAD (foundry CLI), per-template and share_execs
# Result (fresh processes, one noisy box; device open -> templates servable): share_execs LAZY 0.47-0.77 s,
# EAGER 0.65-1.6 s (eager loading of every function of every library in cuLibraryLoadData: restore 0.45-0.65 s
# vs 0.15-0.18 s); per-template LAZY 1.6-8 s, EAGER 1.9-2.4 s. Default (lazy) kept; the bench does not set it.
cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
A=/tmp/foundry_bench_qwen3-235b-a22b/b200
F=paper_2604_06664_b200/foundry
paper_2604_06664_b200/fdy_tool cuda-init 0
for i in 1 2 3; do for opt in "--share-execs" ""; do for m in LAZY EAGER; do
  CUDA_MODULE_LOADING=$m FOUNDRY_DEBUG=1 $F load --archive $A --rank 0 --world 8 $opt > /dev/null 2> /tmp/e.txt
  echo "$m $opt: $(grep -E 'device open|restore done|templates servable' /tmp/e.txt | awk '{print $2}' | tr '\n' ' ')"
done; done; done
