python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --skip-load --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 1 > /dev/null 2>&1
python - <<'PY'
import os, time, json
import paper_2604_06664_b200 as f
A="/tmp/foundry_bench_qwen3-235b-a22b/b200"
for i in range(3):
    t=time.perf_counter(); h=f.load(A, rank=0, world=8); tr=h.replay(1); dt=(time.perf_counter()-t)*1e3
    tm=h.timings(); h.close()
    print(round(dt,1), {k:round(v,1) for k,v in tm.items() if k.endswith('_ms')})
PY
