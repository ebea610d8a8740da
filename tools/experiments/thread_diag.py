import os, sys, threading, time, tempfile
sys.path.insert(0, os.getcwd())
import paper_2604_06664_b200 as foundry
n = int(sys.argv[1])
tmp = tempfile.mkdtemp(); arch = os.path.join(tmp, "a")
foundry.save(foundry.workload_from_text(open(foundry.workload_path("qwen3-235b-a22b")).read()), arch)
for r in range(n): foundry.load(arch, rank=r, world=8, share_execs=True, relocate=True).close()
os.environ["FOUNDRY_DEBUG"] = "1"
b = threading.Barrier(n)
t_all = time.perf_counter()
res = {}
def run(r):
    b.wait(); s = time.perf_counter()
    h = foundry.load(arch, rank=r, world=8, share_execs=True, relocate=True)
    res[r] = ((time.perf_counter() - s) * 1e3, h.timings()); h.close()
ts = [threading.Thread(target=run, args=(r,)) for r in range(n)]
[t.start() for t in ts]; [t.join() for t in ts]
print("makespan", round((time.perf_counter() - t_all) * 1e3, 1))
for r in range(n):
    w, t = res[r]
    print(r, round(w, 1), {k: round(v, 1) for k, v in t.items() if k.endswith("_ms")}, flush=True)
