"""What a launch of this size can reach on this GPU: times torch's own fill and
copy kernels over the member-image size next to the materialize launches
(delta = 0 and delta != 0), all cold-L2, CUDA events on the launching stream.

    python tools/gpu_floor.py [archive_dir]
"""
from __future__ import annotations

import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_06664_b200 import capi  # noqa: E402


def main() -> None:
    arch = sys.argv[1] if len(sys.argv) > 1 else "/tmp/foundry_bench_qwen3-235b-a22b/b200"
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    h = capi.store_header(blob)
    alg = capi.algorithmic_bytes(h)
    n = h["members_image_bytes"]
    api = capi.CApi()
    dev = api.device_open(0)
    store = api.store_upload(dev, blob)
    members, _ = api.materialize(dev, store, 0, 8)
    flush_w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush_r = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")

    def flush():
        flush_w.zero_()
        torch.count_nonzero(flush_r)
        torch.cuda.synchronize()

    def timed(fn, reps=20):
        out = []
        for _ in range(reps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1) * 1e3)
        return {"best_us": min(out), "median_us": statistics.median(out)}

    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    src = torch.ones(n, dtype=torch.uint8, device="cuda")
    res = {
        "member_bytes": n,
        "algorithmic_bytes": alg["total"],
        "torch_fill(write n)": timed(lambda: dst.fill_(7)),
        "torch_copy(read n + write n)": timed(lambda: dst.copy_(src)),
    }
    base = h["old_base"]
    for name, nb in (("materialize delta=0", 0), ("materialize delta=0x10000", base + 0x10000)):
        ks = []
        for _ in range(20):
            flush()
            _, ms = api.materialize(dev, store, 3, 8, nb, members)
            ks.append(ms * 1e3)
        res[name] = {"best_us": min(ks), "median_us": statistics.median(ks)}
    for k, v in res.items():
        if isinstance(v, dict):
            byt = alg["total"] if k.startswith("materialize") else (n if "fill" in k else 2 * n)
            v["GBps_median"] = byt / (v["median_us"] * 1e-6) / 1e9
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
