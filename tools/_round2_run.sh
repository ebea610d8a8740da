cd $GRAFT_REPO_ROOT
python -m pytest tests -x -q -m gpu > gpurun_out/r2_tests.txt 2>&1; tail -3 gpurun_out/r2_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python tools/gpu_thread_vs_process.py 2 > gpurun_out/thread_vs_process2.json 2>&1; tail -c 600 gpurun_out/thread_vs_process2.json
python tools/gpu_thread_vs_process.py 4 > gpurun_out/thread_vs_process4.json 2>&1; tail -c 600 gpurun_out/thread_vs_process4.json
python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 400 gpurun_out/r2_bench.json
bash tools/gpu_profile_bench.sh > gpurun_out/r2_profile.log 2>&1; tail -2 gpurun_out/r2_profile.log
