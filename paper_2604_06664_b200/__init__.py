"""B200-native LOAD path of Foundry (arxiv 2604.06664), drop-in for the
reference's Python surface (reference proj/python/foundry/__init__.py:7-41).

Everything here is backed by the in-tree native build (libfoundry_b200.so +
the `_foundry` pybind11 module); there is no Python or CPU fallback for the
LOAD path, and importing fails loudly if the extension has not been built
(run `python -m paper_2604_06664_b200.build` or `__graft_entry__.build()`).
"""
from __future__ import annotations

import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))

try:
    from ._foundry import (  # noqa: F401
        FoundryError,
        SaveOutcome,
        ServingHandle,
        WorkloadSpec,
        __version__,
        bench,
        cuda_device_count,
        diff_archives,
        inspect_graph_json,
        inspect_text,
        load,
        pack,
        pack_archive,
        preset,
        preset_names,
        save,
        spec_text,
        unpack_archive,
        workload_from_text,
        write_comm_slots,
    )
except ImportError as exc:  # pragma: no cover - exercised only on a broken build
    raise ImportError(
        "paper_2604_06664_b200: the native extension is missing or failed to load "
        f"({exc}); build it with `python -m paper_2604_06664_b200.build`"
    ) from exc

LIBRARY_PATH = _os.path.join(_HERE, "libfoundry_b200.so")
WORKLOADS = _os.path.join(_HERE, "workloads")


def workload_path(name: str) -> str:
    """Path of a bundled tier-R spec (llama3-8b, qwen3-8b, qwen3-30b-a3b, ...)."""
    return _os.path.join(WORKLOADS, name + ".spec")


__all__ = [
    "FoundryError",
    "SaveOutcome",
    "ServingHandle",
    "WorkloadSpec",
    "__version__",
    "bench",
    "cuda_device_count",
    "diff_archives",
    "inspect_graph_json",
    "inspect_text",
    "load",
    "pack",
    "pack_archive",
    "unpack_archive",
    "preset",
    "preset_names",
    "save",
    "spec_text",
    "workload_from_text",
    "workload_path",
    "write_comm_slots",
    "LIBRARY_PATH",
]
