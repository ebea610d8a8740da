python bench.py --skip-load --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 1 > /dev/null 2>&1
A=/tmp/foundry_bench_qwen3-235b-a22b/b200
./paper_2604_06664_b200/fdy_tool instbench $A 2>&1 | grep -E "layered|template"
