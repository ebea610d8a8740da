cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
A=/tmp/foundry_bench_qwen3-235b-a22b/b200
C=paper_2604_06664_b200/foundry
T=paper_2604_06664_b200/fdy_tool
$T cuda-init
for i in 1 2 3; do
  s=$(date +%s%N); $T cuda-init; e=$(date +%s%N); echo "cuda-init $(( (e-s)/1000000 )) ms"
  s=$(date +%s%N); FOUNDRY_DEBUG=1 $C load --archive $A --rank 0 --world 8 --share-execs > /dev/null 2> /tmp/e.txt; e=$(date +%s%N)
  echo "share-execs wall $(( (e-s)/1000000 )) ms"; grep -E "integrity done|restore done|materialize done|group 0:|foreground done" /tmp/e.txt | tr '\n' ' '; echo
done
