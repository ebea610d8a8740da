import os, sys, time, statistics, json
sys.path.insert(0, os.getcwd())
import paper_2604_06664_b200 as f
A = "/tmp/foundry_bench_qwen3-235b-a22b/b200"
h = f.load(A, rank=0, world=8); h.close()  # warm-up
res = {}
for mode in ["overlap", "serial"] * 3:
    if mode == "serial": os.environ["FOUNDRY_EXP_SERIAL_RESTORE"] = "1"
    else: os.environ.pop("FOUNDRY_EXP_SERIAL_RESTORE", None)
    for shared in (False, True):
        t0 = time.perf_counter(); h = f.load(A, rank=0, world=8, share_execs=shared); ms = (time.perf_counter() - t0) * 1e3
        t = h.timings(); h.close()
        res.setdefault((mode, shared), []).append((round(ms), round(t["restore_ms"]), round(t["instantiate_ms"]), round(t.get("function_load_ms", 0))))
for k, v in res.items(): print(k, v)
