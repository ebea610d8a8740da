#!/usr/bin/env python3
"""Headline acceptance (BASELINE config 5): the Qwen3-235B-A22B-shaped TP8 decode
graph set LOADed and replay-verified on every GPU of the node, one process per
GPU, each rank materializing its own TP rank (rank = global rank % 8).

    python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 \\
        --master-addr 127.0.0.1 --master-port 29533 tools/verify_tp8.py [--batches all]

Per rank: foundry.load(archive, rank, 8) (the store reaches peers the same way
the bench does), then every batch (or a sample) is replayed on the device and its
trace compared with the trace derived from the CPU oracle's materialization of
the same rank (oracle/, test infrastructure), plus one fresh-capture check.
Rank 0 prints one JSON line; exit code 0 only if every rank passed.
FOUNDRY_BENCH_SHARED_GPU=1 runs all ranks on cuda:0 (gloo plumbing) for a
one-GPU check of the same code.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main() -> int:
    p = argparse.ArgumentParser()
    p.add_argument("--workload", default="qwen3-235b-a22b")
    p.add_argument("--batches", default="sample", choices=["sample", "all"])
    args = p.parse_args()
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    shared = os.environ.get("FOUNDRY_BENCH_SHARED_GPU") == "1"
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0 if shared else local)
    if world > 1:
        dist.init_process_group("gloo" if shared else "nccl", init_method="env://")
    import bench  # the archive cache and the barrier protocol of the bench
    import fndg
    from oracle_lib import Oracle
    import paper_2604_06664_b200 as foundry

    barrier = (lambda: dist.barrier()) if world > 1 else (lambda: None)
    archive, _ = bench.prepare_archives(args.workload, rank, barrier)
    tp = rank % 8
    t0 = time.perf_counter()
    h = foundry.load(archive, rank=tp, world=8, relocate=shared)
    load_ms = (time.perf_counter() - t0) * 1e3
    base = json.load(open(os.path.join(archive, "manifest")))["allocator"]["base"]
    oracle = Oracle(os.path.join(ROOT, "oracle", "_build", "liboracle.so"))
    container, _ = oracle.materialize_archive(archive, tp, 8, h.region_base() - base)
    hidden = fndg.hidden_map(archive)
    want = {g.label: g for g in fndg.graphs(container)}
    batches = h.batches() if args.batches == "all" else h.batches()[::17] + [h.batches()[-1]]
    bad = [b for b in batches if h.replay(b) != fndg.trace_text(want[b], hidden, oracle.crc64)]
    ok_capture, report = h.fresh_capture_check(batches[len(batches) // 2])
    passed = not bad and ok_capture
    res = {"rank": rank, "tp_rank": tp, "load_ms": load_ms, "replayed": len(batches),
           "mismatches": bad[:5], "fresh_capture": report, "passed": passed}
    h.close()
    results = [None] * world
    if world > 1:
        dist.all_gather_object(results, res)
    else:
        results = [res]
    if rank == 0:
        print(json.dumps({"workload": args.workload, "ranks": world,
                          "all_passed": all(r["passed"] for r in results), "per_rank": results}))
    if world > 1:
        dist.destroy_process_group()
    return 0 if all(r["passed"] for r in results) else 1


if __name__ == "__main__":
    sys.exit(main())
