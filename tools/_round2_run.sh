cd $GRAFT_REPO_ROOT
python -m pytest tests -x -q -m gpu > gpurun_out/r2_tests.txt 2>&1; tail -3 gpurun_out/r2_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --impl reference > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; tail -c 300 gpurun_out/r2_ref.json
python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 400 gpurun_out/r2_bench.json
bash tools/gpu_profile_bench.sh > gpurun_out/r2_profile.log 2>&1; tail -2 gpurun_out/r2_profile.log
ncu --set full --clock-control none --import-source on -k regex:"pack_(walk|images)" -c 2 -o gpurun_out/prof_pack -f python tools/gpu_pack_bench.py qwen3-235b-a22b 1 > /dev/null 2>&1; ls -la gpurun_out/prof_pack.ncu-rep
