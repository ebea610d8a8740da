# e2e: lanes of the early (store) stager. Measured (since-removed FDY_EARLY knob): 4 lanes median 3.85-4.0 ms,
# 6 lanes 4.0, 8 lanes 4.08 (the main thread parsing the manifest loses its core) -> 4 kept.
cd $GRAFT_REPO_ROOT
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
for i in 1 2; do for e in 4 8 6; do REPS=12 TAG="early $e" FDY_EARLY=$e FOUNDRY_DEBUG=1 python tools/experiments/e2e.py 2> gpurun_out/early_$e.txt; tail -1 gpurun_out/early_$e.txt; grep -E "manifest parsed|store verified" gpurun_out/early_$e.txt | tail -4 | tr '\n' ' '; echo; done; done
