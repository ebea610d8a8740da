"""The C-ABI library loads, exports every symbol include/foundry_b200.h
declares, and fails loudly (no CPU fallback) when no GPU is present."""
from __future__ import annotations

import ctypes
import os

import pytest

from conftest import has_gpu


def test_every_declared_function_is_exported(native_build):
    from paper_2604_06664_b200 import capi

    lib = ctypes.CDLL(capi.LIB_PATH)
    names = capi.declared_functions()
    assert "fdy_load" in names and "fdy_materialize" in names and "fdy_prepare_archive" in names
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_version_and_options_defaults(native_build):
    from paper_2604_06664_b200 import capi

    api = capi.CApi()
    assert b"sm_100a" in api.lib.fdy_version()
    o = capi.LoadOptions()
    api.lib.fdy_load_options_init(ctypes.byref(o))
    # reference LoadOptions defaults (pipeline.hpp:80-86)
    assert (o.rank, o.world, o.preallocate, o.prepare_lanes) == (0, 1, 1, 4)
    assert (o.relocate, o.skip_binary_restore, o.base_shift_granules) == (0, 0, 0)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_no_gpu_is_a_loud_error(native_build, archives):
    from paper_2604_06664_b200 import capi

    api = capi.CApi()
    assert api.lib.fdy_device_count() == 0
    arch, _ = archives("micro")
    o = capi.LoadOptions()
    api.lib.fdy_load_options_init(ctypes.byref(o))
    h = ctypes.c_void_p()
    rc = api.lib.fdy_load(arch.encode(), ctypes.byref(o), ctypes.byref(h))
    assert rc == 15  # FDY_ERR_NO_DEVICE
    assert api.lib.fdy_last_error().startswith(b"device-unavailable")
    d = ctypes.c_void_p()
    assert api.lib.fdy_device_open(0, ctypes.byref(d)) == 15


def test_errors_map_onto_the_reference_codes(foundry, tmp_path):
    from paper_2604_06664_b200 import capi

    api = capi.CApi()
    h = ctypes.c_void_p()
    o = capi.LoadOptions()
    api.lib.fdy_load_options_init(ctypes.byref(o))
    o.rank, o.world = 2, 2
    rc = api.lib.fdy_load(str(tmp_path).encode(), ctypes.byref(o), ctypes.byref(h))
    if has_gpu():
        assert rc == 1 and b"rank 2 is outside world size 2" in api.lib.fdy_last_error()
    else:
        assert rc in (1, 15)
