"""GPU-side SAVE to an archive: LOAD an archive for some rank,
stream-capture every batch on the device, extract the driver's graphs, lower
the comm nodes back to stubs and write a reference-layout archive.

The round trip is exact: the new graphs.bin, grouping manifest, catalog and
patch table equal the source archive's byte for byte (captures from rank 3 of
4 and from rank 0 of 1 alike), the reference LOADs it and replays every batch
like the source, and this build LOADs it bit-exactly against the oracle."""
from __future__ import annotations

import json
import os
import subprocess

import pytest

import fndg
from conftest import manifest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _release_handles():
    import gc
    yield
    gc.collect()


@pytest.mark.parametrize("name,rank,world", [("micro", 0, 1), ("llama3-8b", 0, 1), ("moe-spmd", 3, 4)])
def test_save_captured_round_trip(foundry, load, oracle, archives, tmp_path, name, rank, world):
    src, outcome = archives(name)
    out = str(tmp_path / "captured")
    h = load(src, rank=rank, world=world)
    graphs, templates = h.save_captured(out)
    assert (graphs, templates) == (outcome.total_graphs, outcome.template_count)
    h.close()
    for f in ("graphs.bin", "catalog.bin", "patch.bin", "memlayout.bin"):
        assert open(os.path.join(out, f), "rb").read() == open(os.path.join(src, f), "rb").read(), f
    ms, mo = manifest(src), manifest(out)
    assert mo["grouping"] == ms["grouping"]
    assert {k: v for k, v in mo["files"].items() if k != "templates.fdt"} == \
           {k: v for k, v in ms["files"].items() if k != "templates.fdt"}
    # this build LOADs the captured archive bit-exactly (any rank)
    h2 = load(out, rank=1 % world, world=world)
    container, _ = oracle.materialize_archive(out, 1 % world, world)
    hidden = fndg.hidden_map(out)
    want = {g.label: fndg.trace_text(g, hidden, oracle.crc64) for g in fndg.graphs(container)}
    for b in h2.batches()[::5] + [h2.batches()[-1]]:
        assert h2.replay(b) == want[b], "batch %d" % b


def test_save_captured_archive_loads_in_the_reference(foundry, load, archives, tmp_path, ref_tool):
    src, _ = archives("moe-spmd")
    out = str(tmp_path / "captured")
    h = load(src, rank=2, world=4)
    h.save_captured(out)
    h.close()
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    subprocess.run([ref_tool, "load-traces", src, "1", "4", str(a)], check=True)
    subprocess.run([ref_tool, "load-traces", out, "1", "4", str(b)], check=True)
    assert a.read_text() == b.read_text()


def test_save_captured_refuses_a_relocated_load(foundry, load, archives, tmp_path):
    src, _ = archives("micro")
    load(src)  # holds the captured base
    h = load(src, relocate=True)
    with pytest.raises(foundry.FoundryError, match="relocated"):
        h.save_captured(str(tmp_path / "x"))
