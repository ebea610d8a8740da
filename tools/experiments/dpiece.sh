# e2e: piece size of the store (device file) reads, via a since-removed FDY_DPIECE knob.
# Store verified at: 2 MiB 1.01-1.33 ms, 1 MiB 1.07-1.29, 512 KiB 1.28-1.53; e2e medians 4.24 / 4.30-4.34 / 4.32-4.35 -> 2 MiB kept.
cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
for i in 1 2; do for k in 2048 1024 512; do REPS=12 TAG="store piece $k KiB" FDY_DPIECE=$k FOUNDRY_DEBUG=1 python tools/experiments/e2e.py 2> gpurun_out/dp_$k.txt; tail -1 gpurun_out/dp_$k.txt; grep -E "store verified" gpurun_out/dp_$k.txt | tail -6 | awk '{print $2}' | tr '\n' ' '; echo; done; done
