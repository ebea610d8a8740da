cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
A=/tmp/foundry_bench_qwen3-235b-a22b/b200
C=paper_2604_06664_b200/foundry
for flag in "" "--share-execs" "" "--share-execs"; do
  /usr/bin/time -f "wall %e s  $flag" $C load --archive $A --rank 0 --world 8 $flag > /dev/null
done
FOUNDRY_DEBUG=1 $C load --archive $A --rank 0 --world 8 2>&1 | grep -E "group|done|integrity" | head -30
