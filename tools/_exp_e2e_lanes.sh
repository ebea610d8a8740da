cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
for l in 4 6 8 10 12 16; do echo "rest lanes $l"; FOUNDRY_EXP_REST_LANES=$l python tools/_exp_e2e.py 2>&1 | tail -3 | python -c "
import sys,ast
for line in sys.stdin: d=ast.literal_eval(line); print(' total', d['total_ms'], 'read', d['read_ms'], 'd2h', d['d2h_ms'])"; done
