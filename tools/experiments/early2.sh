# After the fast manifest reader (manifest parsed at ~0.42 ms instead of ~0.78): store stager on 4 / 6 / 8
# lanes -> e2e medians 4.24-4.60 / 4.31-4.35 / 4.39-4.48 ms on this box; the host hashing chain (read_ms 3.3-3.9)
# is the bound, not the store. 4 kept (FDY_EARLY knob removed).
cd $GRAFT_REPO_ROOT
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --skip-load --no-cpu-baseline > /dev/null 2>&1
for i in 1 2; do for e in 4 6 8; do REPS=12 TAG="early $e" FDY_EARLY=$e FOUNDRY_DEBUG=1 python tools/experiments/e2e.py 2> gpurun_out/early_$e.txt; tail -1 gpurun_out/early_$e.txt; grep -E "manifest parsed|store verified" gpurun_out/early_$e.txt | tail -4 | awk '{print $2}' | tr '\n' ' '; echo; done; done
