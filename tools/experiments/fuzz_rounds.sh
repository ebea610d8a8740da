# Extra rounds of the GPU packer / C-ABI fuzzers (seeds beyond the suite's own):
#   FUZZ_ROUNDS="4 5 6" FUZZ_N=150 bash tools/experiments/fuzz_rounds.sh
cd $GRAFT_REPO_ROOT
for R in ${FUZZ_ROUNDS:-4 5 6}; do
  echo "round $R: $(FOUNDRY_FUZZ_ROUND=$R FOUNDRY_FUZZ_N=${FUZZ_N:-150} timeout 900 python -m pytest tests/test_gpu_pack.py tests/test_gpu_capi.py -q -k fuzz -rf 2>&1 | grep -E 'passed|failed|FAILED|Error' | tail -4)"
done
