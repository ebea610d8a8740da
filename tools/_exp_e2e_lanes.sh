cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
for i in 1 2; do for r in 16 12; do
REPS=10 TAG="mmap  $r" FDY_REST_LANES=$r python tools/_exp_e2e.py
REPS=10 TAG="pread $r" FDY_NO_MMAP=1 FDY_REST_LANES=$r python tools/_exp_e2e.py
done; done
