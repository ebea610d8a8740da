# host read / hash throughput of the headline archive's largest file, by thread count
cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
g++ -O2 -std=c++20 -pthread -Ipaper_2604_06664_b200/csrc/include tools/experiments/hashbench.cpp paper_2604_06664_b200/csrc/host/support.cpp -o /tmp/hb
A=/tmp/foundry_bench_qwen3-235b-a22b/b200
for t in 1 4 8 12 16; do /tmp/hb $A/graphs.bin $t | sort | awk '{print}' | tail -9 | grep -v "^$" | sort -u | head -9; done
