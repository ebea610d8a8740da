"""bench.py's N>1 path (one process per rank, store fan-out over CUDA IPC or
a pipelined chain, max-over-ranks timing) on the single test GPU:
FOUNDRY_BENCH_SHARED_GPU=1 puts every rank on cuda:0 with gloo plumbing (NCCL
refuses two ranks on one device). The driver's 8-GPU runs use the same code
with one GPU per rank."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("fanout,n", [("ipc", 2), ("host", 2), ("chain", 2), ("chain", 8), ("ipc", 8)])
def test_bench_n_ranks(native_build, fanout, n):
    """n = 8: the driver's 8-GPU command line, all ranks on the one GPU."""
    env = dict(os.environ, FOUNDRY_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", str(n), "--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--skip-load",
           "--no-cpu-baseline", "--workload", "llama3-8b", "--fanout", fanout]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["scaling"] == "weak" and d["value"] > 0
    assert d["roofline"]["achieved"] > 0 and d["e2e"]["value"] > 0
    assert d["fanout"]["mode"] == fanout
    assert set(d["fanout"]["modes_ms"]) == {"ipc", "chain", "host"}  # all three options
    assert all(v > 0 for v in d["fanout"]["modes_ms"].values())
