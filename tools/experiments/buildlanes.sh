cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
A=/tmp/foundry_bench_qwen3-235b-a22b/b200
T=paper_2604_06664_b200/fdy_tool
$T load $A 0 8 > /dev/null 2>&1
for l in 1 2 4 1 2 4; do echo "lanes $l"; FOUNDRY_BUILD_LANES=$l $T load $A 0 8 2>&1 | grep loaded; done
