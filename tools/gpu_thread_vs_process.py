"""Driver contention: N LOADs of the headline archive at once,
from N threads of one process vs N processes, all on cuda:0. With one GPU
this isolates the host/driver side of an 8-GPU LOAD: inside one process the
CUDA driver serializes graph construction and function loads behind
process-wide locks; separate processes (bench.py's one process per GPU) do
not share them. Every LOAD relocates (relocate=True): concurrent LOADs in one
process cannot all map the captured VA range (one address space), which is
itself a reason for one process per GPU.

    python tools/gpu_thread_vs_process.py [N] [workload]     (prints one JSON line)
"""
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(arch: str, rank: int, go: str) -> None:
    import paper_2604_06664_b200 as foundry
    h = foundry.load(arch, rank=rank, world=8, share_execs=True, relocate=True)  # warm this process (context, pools)
    h.close()
    open(go + ".ready%d" % rank, "w").close()
    while not os.path.exists(go):
        time.sleep(0.001)
    t0 = time.perf_counter()
    h = foundry.load(arch, rank=rank, world=8, share_execs=True, relocate=True)
    wall = (time.perf_counter() - t0) * 1e3
    t = h.timings()
    h.close()
    print(json.dumps({"rank": rank, "wall_ms": wall, "t0": t0, "t1": t0 + wall / 1e3,
                      "instantiate_ms": t["instantiate_ms"], "function_load_ms": t["function_load_ms"],
                      "restore_ms": t["restore_ms"], "build_ms": t["build_ms"]}))


def main() -> None:
    if sys.argv[1:2] == ["child"]:
        child(sys.argv[2], int(sys.argv[3]), sys.argv[4])
        return
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    name = sys.argv[2] if len(sys.argv) > 2 else "qwen3-235b-a22b"
    import paper_2604_06664_b200 as foundry
    tmp = tempfile.mkdtemp()
    arch = os.path.join(tmp, "a")
    foundry.save(foundry.workload_from_text(open(foundry.workload_path(name)).read()), arch)
    out = {"workload": name, "n": n}

    # one LOAD alone (warm process)
    foundry.load(arch, rank=0, world=8, share_execs=True, relocate=True).close()
    t0 = time.perf_counter()
    foundry.load(arch, rank=0, world=8, share_execs=True, relocate=True).close()
    out["alone_ms"] = (time.perf_counter() - t0) * 1e3

    # N threads of this process
    for r in range(n):
        foundry.load(arch, rank=r, world=8, share_execs=True, relocate=True).close()
    walls = [0.0] * n
    barrier = threading.Barrier(n + 1)

    def run(r):
        barrier.wait()
        s = time.perf_counter()
        foundry.load(arch, rank=r, world=8, share_execs=True, relocate=True).close()
        walls[r] = (time.perf_counter() - s) * 1e3

    ths = [threading.Thread(target=run, args=(r,)) for r in range(n)]
    for t in ths:
        t.start()
    t0 = time.perf_counter()
    barrier.wait()
    for t in ths:
        t.join()
    out["threads"] = {"makespan_ms": (time.perf_counter() - t0) * 1e3, "per_load_ms": walls}

    # N processes
    go = os.path.join(tmp, "go")
    procs = [subprocess.Popen([sys.executable, __file__, "child", arch, str(r), go], stdout=subprocess.PIPE,
                              text=True) for r in range(n)]
    while not all(os.path.exists(go + ".ready%d" % r) for r in range(n)):
        time.sleep(0.01)
    open(go, "w").close()
    rows = [json.loads(p.communicate()[0].strip().splitlines()[-1]) for p in procs]
    out["processes"] = {"makespan_ms": (max(r["t1"] for r in rows) - min(r["t0"] for r in rows)) * 1e3,
                        "per_load_ms": [r["wall_ms"] for r in rows],
                        "instantiate_ms": [r["instantiate_ms"] for r in rows],
                        "function_load_ms": [r["function_load_ms"] for r in rows]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
