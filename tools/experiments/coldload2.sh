# Fresh-process LOAD timelines (FOUNDRY_DEBUG), share_execs, 4 rounds, next to context-only processes
cd "$(dirname "$0")/../.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --skip-tier-s --no-cpu-baseline > gpurun_out/coldload_bench.log 2>&1 || tail -5 gpurun_out/coldload_bench.log
A=/tmp/foundry_bench_qwen3-235b-a22b/b200
F=paper_2604_06664_b200/foundry
$F load --archive $A --rank 0 --world 8 --share-execs > /dev/null 2>&1
for i in 1 2 3 4; do
  echo "== round $i"
  s=$(date +%s%N); paper_2604_06664_b200/fdy_tool cuda-init 0 > /dev/null; e=$(date +%s%N); echo "cuda-init wall $(( (e - s) / 1000000 )) ms"
  s=$(date +%s%N)
  FOUNDRY_DEBUG=1 $F load --archive $A --rank 0 --world 8 --share-execs > /tmp/o.txt 2> /tmp/e.txt
  e=$(date +%s%N); echo "load wall $(( (e - s) / 1000000 )) ms"
  grep -v "group \|build group\|built group\|instantiated group" /tmp/e.txt | head -40
done
