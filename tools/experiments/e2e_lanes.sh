# e2e host-lane split. Measured with (since removed) env knobs for the rest stager's
# lane count and nice level: 12 lanes/nice 0 median 4.6-4.75 ms (max 6.2), 16/0 4.26-4.37
# (max 5.8), 16/10 4.42-5.14, 12/10 4.29-4.47, 16/19 4.19-4.31 (max 4.4-5.2) -> 16/19 shipped.
cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
for i in 1 2; do REPS=12 TAG="shipped" python tools/experiments/e2e.py; done
