"""Edge-shaped graph sets through the full LOAD path, in both archive layouts
(B200 store, and the reference's layout packed on the GPU at LOAD): a single
captured graph with one kernel per layer and one layer (the smallest spec the
reference accepts, workload_gen.cpp:87-120), a set where every batch size is its
own template (no member ever differs from a template, so no diffs), one where
every batch size shares a single template, and a small SPMD set patched for
rank 1 of 2. Every batch replays like the C oracle's
materialization, and the counters follow the reference's contract.
"""
from __future__ import annotations

import os

import pytest

import fndg

pytestmark = pytest.mark.gpu

EDGES = {
    # name: (preset, overrides, rank, world)
    "one-graph": ("micro", dict(batch_max=1, thresholds=[], layers=1, kernels_per_layer=1), 0, 1),
    "every-batch-a-template": ("micro", dict(batch_max=5, thresholds=[2, 3, 4, 5]), 0, 1),
    "one-template": ("micro", dict(batch_max=4, thresholds=[]), 0, 1),
    "spmd-six-graphs": ("moe-spmd", dict(batch_max=6, thresholds=[3, 5], layers=1), 1, 2),
}


@pytest.fixture(autouse=True)
def _release_handles():
    import gc
    yield
    gc.collect()


@pytest.mark.parametrize("layout", ["b200", "reference"])
@pytest.mark.parametrize("name", sorted(EDGES))
def test_edge_graph_sets_replay_like_the_oracle(foundry, load, oracle, tmp_path, name, layout):
    preset, overrides, rank, world = EDGES[name]
    spec = foundry.preset(preset)
    for k, v in overrides.items():
        setattr(spec, k, v)
    arch = os.path.join(str(tmp_path), name)
    outcome = foundry.save(spec, arch, b200_artifacts=(layout == "b200"))
    assert outcome.total_graphs == spec.batch_max
    container, _ = oracle.materialize_archive(arch, rank, world)
    hidden = fndg.hidden_map(arch)
    want = {g.label: fndg.trace_text(g, hidden, oracle.crc64) for g in fndg.graphs(container)}
    h = load(arch, rank=rank, world=world)
    assert h.batches() == list(range(1, spec.batch_max + 1))
    for b in h.batches():
        assert h.replay(b) == want[b], "batch %d" % b
    c = h.counters()
    assert c["exec.instantiate_calls"] == outcome.template_count
    assert c["exec.update_calls"] == outcome.total_graphs - outcome.template_count
    ok, report = h.fresh_capture_check(h.batches()[-1])
    assert ok, report


@pytest.fixture(scope="module")
def api(foundry):
    from paper_2604_06664_b200 import capi
    return capi.CApi()


@pytest.fixture(scope="module")
def dev(api):
    d = api.device_open(0)
    yield d
    api.lib.fdy_device_close(d)


@pytest.mark.parametrize("delta", [0, 0x10000])
@pytest.mark.parametrize("name", sorted(EDGES))
def test_edge_graph_sets_prepare_like_the_oracle(foundry, oracle, api, dev, tmp_path, name, delta):
    """fdy_prepare_archive (files -> GPU integrity -> fused kernel -> host memory)
    on both layouts of each edge set, relocated or not, equals the oracle's
    parse_graph_at + relocation + rank patch of every member."""
    import ctypes
    import json

    from paper_2604_06664_b200 import capi
    preset, overrides, rank, world = EDGES[name]
    spec = foundry.preset(preset)
    for k, v in overrides.items():
        setattr(spec, k, v)
    b200, plain = os.path.join(str(tmp_path), "b200"), os.path.join(str(tmp_path), "plain")
    foundry.save(spec, b200)
    foundry.save(spec, plain, b200_artifacts=False)
    base = json.load(open(os.path.join(b200, "manifest")))["allocator"]["base"]
    size = capi.store_header(open(os.path.join(b200, "templates.fdt"), "rb").read())["members_image_bytes"]
    want, _ = oracle.materialize_archive(b200, rank, world, delta)
    for arch in (b200, plain):
        host = api.host_alloc(dev, size)
        try:
            t = api.prepare_archive(dev, arch, rank, world, base + delta if delta else 0, 4, host, size)
            arena = ctypes.string_at(host, t["member_bytes"])
        finally:
            api.lib.fdy_host_free(host)
        assert t["graphs"] == spec.batch_max and t["member_bytes"] == size
        assert foundry._foundry._decode_member_images(b200, arena) == want, arch
