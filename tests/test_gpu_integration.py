"""The drop-in proven with the reference's own pipeline: INTEGRATION.md §2
(oracle/_ref/prepare_fn_demo, the reference LOAD sequence with its PrepareFn
replaced by the GPU materialization through the C-ABI) replays every batch
exactly like the reference's unmodified load() (ref_tool load-traces)."""
from __future__ import annotations

import os
import shutil
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

DEMO = os.path.join(ROOT, "oracle", "_ref", "prepare_fn_demo")


@pytest.mark.parametrize("name,rank,world", [("llama3-8b", 0, 1), ("moe-spmd", 3, 4), ("moe-spmd", 7, 8)])
def test_reference_pipeline_with_the_gpu_prepare_fn(archives, ref_tool, tmp_path, name, rank, world):
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/prepare_fn_demo not built")
    arch, _ = archives(name)
    got, want = tmp_path / "gpu.txt", tmp_path / "ref.txt"
    r = subprocess.run([DEMO, arch, str(rank), str(world), str(got)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    subprocess.run([ref_tool, "load-traces", arch, str(rank), str(world), str(want)], check=True, timeout=600)
    assert got.read_text() == want.read_text()
    assert got.read_text().count("# batch") or len(got.read_text()) > 0


def test_reference_written_archive_through_the_gpu_prepare_fn(archives, ref_tool, tmp_path):
    """An archive the reference itself saved (no B200 artefacts): fdy_load_members
    packs it on the host, the kernel materializes it, the reference replays it."""
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/prepare_fn_demo not built")
    arch = str(tmp_path / "refsave")
    subprocess.run([ref_tool, "save", "moe-spmd", arch], check=True, capture_output=True)
    got, want = tmp_path / "gpu.txt", tmp_path / "ref.txt"
    r = subprocess.run([DEMO, arch, "1", "2", str(got)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    subprocess.run([ref_tool, "load-traces", arch, "1", "2", str(want)], check=True)
    assert got.read_text() == want.read_text()
