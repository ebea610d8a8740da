# Fresh-process LOAD timelines (FOUNDRY_DEBUG) for per-template and share_execs, incl. teardown
cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > gpurun_out/coldload_bench.log 2>&1 || tail -5 gpurun_out/coldload_bench.log
A=/tmp/foundry_bench_qwen3-235b-a22b/b200
F=paper_2604_06664_b200/foundry
$F load --archive $A --rank 0 --world 8 > /dev/null 2>&1
for opt in "--share-execs" "" "--share-execs" "--no-prealloc --share-execs"; do
  echo "== load $opt"
  s=$(date +%s%N)
  FOUNDRY_DEBUG=1 $F load --archive $A --rank 0 --world 8 $opt > /tmp/o.txt 2> /tmp/e.txt
  e=$(date +%s%N); echo "wall $(( (e - s) / 1000000 )) ms"
  grep -v "group \|build group\|built group\|instantiated group" /tmp/e.txt
done
paper_2604_06664_b200/fdy_tool cuda-init 0
for i in 1 2; do s=$(date +%s%N); paper_2604_06664_b200/fdy_tool cuda-init 0; e=$(date +%s%N); echo "cuda-init wall $(( (e - s) / 1000000 )) ms"; done
