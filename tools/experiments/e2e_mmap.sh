cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
for v in "" "FOUNDRY_EXP_MMAP=1" "" "FOUNDRY_EXP_MMAP=1"; do echo "== $v"; env $v python tools/experiments/e2e.py 2>&1 | tail -3 | python -c "
import sys,ast
for line in sys.stdin: d=ast.literal_eval(line); print(' total', d['total_ms'], 'read', d['read_ms'])"; done
