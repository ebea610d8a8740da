"""Does a resident CUDA context (another process holding the device, as a
serving box with the persistence daemon or any running job has) change the
cost of creating a context in a fresh process? Times `fdy_tool cuda-init`
(exec to its 'ready' line) N times with nothing else on the GPU, then N times
while `fdy_tool cuda-hold` keeps a context open. Prints one JSON line."""
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
TOOL = os.path.join(ROOT, "paper_2604_06664_b200", "fdy_tool")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 6


def once():
    t0 = time.perf_counter()
    p = subprocess.Popen([TOOL, "cuda-init", "0"], stdout=subprocess.PIPE, text=True)
    t = None
    for line in p.stdout:
        if t is None and "ready" in line:
            t = time.perf_counter()
    p.wait()
    return (t - t0) * 1e3


def load_once(archive):
    t0 = time.perf_counter()
    p = subprocess.Popen([os.path.join(ROOT, "paper_2604_06664_b200", "foundry"), "load", "--archive", archive,
                          "--rank", "0", "--world", "8", "--device", "0", "--share-execs"],
                         stdout=subprocess.PIPE, text=True)
    t = None
    for line in p.stdout:
        if t is None and " ready: " in line:
            t = time.perf_counter()
    p.wait()
    return (t - t0) * 1e3


def stat(xs):
    return {"median": statistics.median(xs), "min": min(xs), "max": max(xs), "n": len(xs)}


pm = subprocess.run(["nvidia-smi", "--query-gpu=persistence_mode", "--format=csv,noheader"],
                    capture_output=True, text=True).stdout.strip()
sys.path.insert(0, ROOT)
from bench import prepare_archives  # noqa: E402

archive, _ = prepare_archives("qwen3-235b-a22b", 0, lambda: None)
once()
alone, load_alone = [], []
for _ in range(N):
    time.sleep(1.0)
    alone.append(once())
    time.sleep(1.0)
    load_alone.append(load_once(archive))
hold = subprocess.Popen([TOOL, "cuda-hold", "0"], stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)
hold.stdout.readline()
held, load_held = [], []
for _ in range(N):
    time.sleep(1.0)
    held.append(once())
    time.sleep(1.0)
    load_held.append(load_once(archive))
hold.stdin.close()
hold.wait()
print(json.dumps({"persistence_mode": pm, "cuda_init_alone_ms": stat(alone), "cuda_init_while_held_ms": stat(held),
                  "load_share_execs_alone_ms": stat(load_alone), "load_share_execs_while_held_ms": stat(load_held),
                  "alone": alone, "held": held}))
