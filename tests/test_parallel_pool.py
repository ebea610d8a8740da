"""The host worker pool behind foundry::parallel_for (include/foundry/parallel.hpp):
results, exception propagation, nested and concurrent calls, fork safety."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "paper_2604_06664_b200", "csrc", "include")


@pytest.mark.skipif(shutil.which("g++") is None, reason="no host compiler")
def test_parallel_for_pool(tmp_path):
    exe = tmp_path / "pool_check"
    subprocess.run(["g++", "-std=c++20", "-O2", "-pthread", "-I", INC,
                    os.path.join(ROOT, "tests", "native", "parallel_pool_check.cpp"), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stdout + out.stderr
