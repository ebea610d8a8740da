"""Shared fixtures.

`-m "not gpu"` tests run in the CPU-only container: the oracle against the
reference's golden vectors / the compiled reference, the SAVE writer, the
template-store packer (through a NumPy emulation of the kernel), the C-ABI
exports and the multi-process host logic (gloo). `-m gpu` tests are the
parity tests proper on a B200 and go through the native library.
"""
from __future__ import annotations

import ctypes
import json
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.join(ROOT, "tests")
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
FDY_TOOL = os.path.join(ROOT, "paper_2604_06664_b200", "fdy_tool")
WORKLOADS = os.path.join(ROOT, "paper_2604_06664_b200", "workloads")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def native_build():
    """Build the native library and the oracle once per session (no-op when fresh)."""
    from paper_2604_06664_b200 import build as b

    b.build()
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    return True


@pytest.fixture(scope="session")
def foundry(native_build):
    import paper_2604_06664_b200 as f

    return f


@pytest.fixture(scope="session")
def oracle(native_build):
    from oracle_lib import Oracle

    return Oracle(ORACLE_SO)


@pytest.fixture(scope="session")
def ref_tool():
    if not os.path.exists(REF_TOOL):
        pytest.skip("oracle/_ref/ref_tool not built (needs /root/reference)")
    return REF_TOOL


def spec_path(name: str) -> str:
    p = os.path.join(WORKLOADS, name + ".spec")
    return p if os.path.exists(p) else name


@pytest.fixture(scope="session")
def archives(tmp_path_factory, foundry):
    """Session cache of archives written by this build's SAVE (with B200 artefacts)."""
    root = tmp_path_factory.mktemp("archives")
    cache = {}

    def get(name: str, b200: bool = True) -> str:
        key = (name, b200)
        if key not in cache:
            out = os.path.join(str(root), name + ("" if b200 else "-plain"))
            spec = foundry.workload_from_text(open(spec_path(name)).read()) if os.path.exists(
                spec_path(name)) else foundry.preset(name)
            outcome = foundry.save(spec, out, b200_artifacts=b200)
            cache[key] = (out, outcome)
        return cache[key]

    return get


def manifest(path: str) -> dict:
    with open(os.path.join(path, "manifest")) as f:
        return json.load(f)


def has_gpu() -> bool:
    try:
        import paper_2604_06664_b200 as f

        return f.cuda_device_count() > 0
    except Exception:
        return False


@pytest.fixture
def load(foundry):
    """foundry.load that closes every handle it returned at test teardown."""
    handles = []

    def _load(*args, **kwargs):
        h = foundry.load(*args, **kwargs)
        handles.append(h)
        return h

    yield _load
    for h in handles:
        h.close()
