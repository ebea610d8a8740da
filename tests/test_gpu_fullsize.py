"""Full-size replay verification of every BASELINE config (BASELINE.json
configs 1-5 at their tier-R sizes): LOAD through the public API
for the (rank, world) each config is quoted on, replay against the oracle's
traces, and check that the materialized graphs reproduce freshly captured
graphs (north_star correctness clause; reference acceptance criteria 1 and 8,
acceptance.cpp:108-141,373-415).

Per handle: one batch of every template, every 16th label and the last label
are replayed and device-verified; one fresh-capture equivalence per template
on the first rank of each config. The headline set (config 5) replays all
512 batches on all 8 TP ranks, the ranks sharing this GPU: rank 0 lands at
the captured base, ranks 1-7 are relocated (K1) while rank 0 holds it.
"""
from __future__ import annotations

import os

import pytest

import fndg
from conftest import manifest

pytestmark = pytest.mark.gpu

LANES = max(4, os.cpu_count() or 4)


@pytest.fixture(autouse=True)
def _release_handles():
    import gc
    yield
    gc.collect()


def expected(oracle, arch, rank, world, delta=0):
    container, _ = oracle.materialize_archive(arch, rank, world, delta, LANES)
    hidden = fndg.hidden_map(arch)
    return {g.label: fndg.trace_text(g, hidden, oracle.crc64) for g in fndg.graphs(container)}


def template_firsts(arch):
    return [g["locators"][0][0] for g in manifest(arch)["grouping"]["groups"]]


def sample(arch, labels):
    picked = set(template_firsts(arch)) | set(labels[::16]) | {labels[-1]}
    return sorted(picked)


# (workload, world, ranks, share_execs): the (rank, world) each BASELINE config is quoted on
CONFIGS = [
    ("llama3-8b", 1, [0], False),            # config 1: TP=1, 35 capture sizes
    ("qwen3-8b", 1, [0], False),             # config 2: dense TP=1, 512 graphs / 20 templates
    ("qwen3-30b-a3b", 1, [0], False),        # config 3: MoE on 1 ...
    ("qwen3-30b-a3b", 2, [0, 1], True),      #           ... and 2 GPUs
    ("llama3-70b", 4, [0, 1, 2, 3], True),   # config 4: TP=4 ...
    ("llama3-70b", 8, list(range(8)), True), #           ... and TP=8 from one capture
]


@pytest.mark.parametrize("name,world,ranks,share", CONFIGS,
                         ids=["%s-w%d" % (c[0], c[1]) for c in CONFIGS])
def test_baseline_config_full_size_replay_verified(foundry, load, oracle, archives, name, world, ranks, share):
    arch, outcome = archives(name)
    base = manifest(arch)["allocator"]["base"]
    handles = []
    for rank in ranks:
        # every rank of the config at once on this one GPU: the first one holds
        # the captured base, the others are relocated onto their own regions
        h = load(arch, rank=rank, world=world, relocate=True, share_execs=share, prepare_lanes=LANES)
        handles.append(h)
        delta = h.region_base() - base
        assert (delta != 0) == (rank != ranks[0])
        want = expected(oracle, arch, rank, world, delta)
        labels = h.batches()
        assert labels == sorted(want) and len(labels) == outcome.total_graphs
        for b in sample(arch, labels):
            assert h.replay(b) == want[b], "%s rank %d/%d batch %d" % (name, rank, world, b)
        if rank == ranks[0]:
            for b in template_firsts(arch):
                ok, report = h.fresh_capture_check(b)
                assert ok, "%s batch %d: %s" % (name, b, report)


def test_headline_tp8_every_rank_every_batch(foundry, load, oracle, archives):
    """Config 5, the paper's headline case: the qwen3-235b-a22b~ TP8 decode set
    (512 graphs x 1036 nodes, 12 templates). All 8 TP ranks are LOADed from the
    one single-GPU capture (rank/world + comm kernel patching), every one of
    the 8 x 512 graphs is replayed and device-verified against the oracle, and
    rank 0 reproduces a fresh capture of every template."""
    arch, outcome = archives("qwen3-235b-a22b")
    base = manifest(arch)["allocator"]["base"]
    assert outcome.total_graphs == 512 and outcome.template_count == 12
    handles = []
    for rank in range(8):
        h = load(arch, rank=rank, world=8, relocate=True, share_execs=True, prepare_lanes=LANES)
        handles.append(h)
        delta = h.region_base() - base
        want = expected(oracle, arch, rank, 8, delta)
        for b in h.batches():
            assert h.replay(b) == want[b], "rank %d batch %d" % (rank, b)
        if rank == 0:
            assert delta == 0
            for b in template_firsts(arch):
                ok, report = h.fresh_capture_check(b)
                assert ok, "batch %d: %s" % (b, report)
    assert len({h.region_base() for h in handles}) == 8
