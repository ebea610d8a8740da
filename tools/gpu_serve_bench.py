"""Serve-path timing (A12): one LOAD of the headline archive per mode, then
serve() of every batch in label order; prints us per serve. With
device_updates the per-serve work is one fdy_serve_kernel launch (profiled by
tools/gpu_profile_bench.sh).

    python tools/gpu_serve_bench.py [archive_dir]
"""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_06664_b200 as foundry  # noqa: E402
import torch  # noqa: E402  (device-wide synchronize around the sweep)


def main() -> None:
    arch = sys.argv[1] if len(sys.argv) > 1 else "/tmp/foundry_bench_qwen3-235b-a22b/b200"
    modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["per_template", "device_updates"]
    out = {}
    for mode in modes:
        h = foundry.load(arch, rank=0, world=8, device_updates=mode == "device_updates",
                         share_execs=mode == "shared_execs")
        bs = h.batches()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for b in bs:
            h.serve(b)
        host_ms = (time.perf_counter() - t0) * 1e3
        torch.cuda.synchronize()  # device_updates queues its serve kernels
        ms = (time.perf_counter() - t0) * 1e3
        out[mode] = {"serves": len(bs), "us_per_serve": ms * 1e3 / len(bs),
                     "host_us_per_serve": host_ms * 1e3 / len(bs)}
        h.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
