"""bench.py --impl reference runs on CPU (the reference's own save + CPU
materialization timing through oracle/_ref/ref_tool): its JSON line keeps the
contract the driver parses, prints the same `config` as our arm, and never
imports this build's package or loads its libraries."""
from __future__ import annotations

import json
import os
import subprocess
import sys

from conftest import ROOT

_RUN = """
import runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1", "--workload", "llama3-8b"]
runpy.run_path("bench.py", run_name="__main__")
bad = [m for m in sys.modules if m.startswith(("paper_2604_06664_b200", "foundry"))]
maps = open("/proc/self/maps").read()
bad += [l.split()[-1] for l in maps.splitlines() if "libfoundry_b200" in l or "_foundry" in l]
print("LEAKED", sorted(set(bad)))
"""


def test_reference_arm_line(native_build, ref_tool):
    r = subprocess.run([sys.executable, "-c", _RUN], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "ms" and d["higher_is_better"] is False
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["cpu_model"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]
    assert d["full_load"]["value"] > 0 and d["serve_replay_all"]["batches"] == 35
    assert "LEAKED []" in r.stdout, r.stdout[-500:]
    # the same config dict our arm prints (bench_config over the same archive bytes)
    sys.path.insert(0, ROOT)
    import bench

    plain = bench.reference_archive("llama3-8b")
    assert d["config"] == bench.bench_config("llama3-8b", plain, 0)
    assert d["config"]["graphs"] == 35 and d["config"]["nodes"] == 35 * 258
