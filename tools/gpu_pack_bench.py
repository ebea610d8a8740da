"""GPU packer vs offline packer on a reference-written archive of a BASELINE
config: phase timings of pack_template_store_device (graphs.bin already read),
the CPU packer on all host threads, and store equality.
Usage: python tools/gpu_pack_bench.py [workload] [reps]"""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_06664_b200 as foundry  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-235b-a22b"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
with tempfile.TemporaryDirectory() as tmp:
    arch = os.path.join(tmp, "plain")
    foundry.save(foundry.workload_from_text(open(foundry.workload_path(name)).read()), arch, b200_artifacts=False)
    rows = []
    for r in range(reps):
        gpu, t = foundry._foundry._pack_store_bytes(arch, True)
        rows.append(t)
    t0 = time.perf_counter()
    cpu, _ = foundry._foundry._pack_store_bytes(arch, False)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    best = min(rows, key=lambda t: t["total_ms"])
    print(json.dumps({"workload": name, "store_bytes": len(gpu), "equal": gpu == cpu,
                      "gpu_pack": best, "gpu_total_ms_all": [round(t["total_ms"], 3) for t in rows],
                      "cpu_pack_ms_incl_reads": round(cpu_ms, 1), "host_threads": os.cpu_count()}))
