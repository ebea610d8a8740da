"""INTEGRATION.md §2 is compiled, not illustrated: `make -C oracle ref`
extracts its C++ block verbatim and links it against the unmodified reference
(oracle/_ref/libfoundry_core.a) and this build's C-ABI (include/foundry_b200.hpp
over libfoundry_b200.so). Here (no GPU) it must build and fail cleanly with
device-unavailable; tests/test_gpu_integration.py runs it on a B200."""
from __future__ import annotations

import os
import subprocess
import sys

from conftest import ROOT

DEMO = os.path.join(ROOT, "oracle", "_ref", "prepare_fn_demo")


def test_integration_block_compiles_against_the_reference(ref_tool, tmp_path, archives):
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    src = open(os.path.join(ROOT, "oracle", "_ref", "prepare_fn_demo.cpp")).read()
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    assert src.strip() in doc  # verbatim
    assert "foundry_b200::GpuPrepare" in src and "ServingSet::build" in src
    assert os.path.getmtime(DEMO) >= os.path.getmtime(os.path.join(ROOT, "INTEGRATION.md"))
    import paper_2604_06664_b200 as foundry
    if foundry.cuda_device_count() == 0:
        arch, _ = archives("micro")
        r = subprocess.run([DEMO, arch, "0", "1", str(tmp_path / "t.txt")], capture_output=True, text=True)
        assert r.returncode == 15, (r.returncode, r.stderr)  # FDY_ERR_NO_DEVICE
        assert "device-unavailable" in r.stderr


def test_cxx_header_compiles_standalone(tmp_path):
    """include/foundry_b200.hpp needs nothing but include/ and the .so."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "foundry_b200.hpp"\nint main() { return fdy_device_count() < 0; }\n')
    lib = os.path.join(ROOT, "paper_2604_06664_b200")
    r = subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src),
                        "-L" + lib, "-lfoundry_b200", "-Wl,-rpath," + lib, "-o", str(tmp_path / "t")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(tmp_path / "t")]).returncode == 0
