"""GPU parity of the full LOAD path (reference pipeline.cpp:447-569 semantics).

Every replayed trace is compared with the trace derived from the C oracle's
materialization of the same member (parse_graph_at + relocation + rank patch),
and the oracle itself is pinned to the reference in test_oracle.py.
"""
from __future__ import annotations

import os
import shutil

import pytest

import fndg
from conftest import manifest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _release_handles():
    """Handles own a VA reservation at the captured base; release every handle
    a test created (even when it failed) before the next test loads."""
    import gc
    yield
    gc.collect()


def expected_traces(oracle, archive, rank=0, world=1, delta=0):
    container, _ = oracle.materialize_archive(archive, rank, world, delta)
    hidden = fndg.hidden_map(archive)
    return {g.label: fndg.trace_text(g, hidden, oracle.crc64) for g in fndg.graphs(container)}


@pytest.mark.parametrize("name", ["micro", "llama3-8b", "moe-spmd"])
def test_load_replays_every_batch_like_the_oracle(foundry, load, oracle, archives, name):
    arch, outcome = archives(name)
    h = load(arch)
    assert h.batches() == list(range(1, outcome.total_graphs + 1))
    want = expected_traces(oracle, arch)
    for b in h.batches():
        assert h.replay(b) == want[b], "batch %d" % b
    c = h.counters()
    assert c["exec.instantiate_calls"] == outcome.template_count
    assert c["capture.begin_calls"] == 0
    assert c["catalog.prelink_calls"] == 0
    assert c["replay.launch_calls"] == outcome.total_graphs
    # one on-demand update per non-template member (test_smoke.py:43, acceptance criterion 5)
    assert c["exec.update_calls"] == outcome.total_graphs - outcome.template_count


def test_save_traces_equal_load_traces_at_world_one(foundry, load, archives):
    arch, outcome = archives("micro")
    h = load(arch)
    for b in h.batches():
        assert h.replay(b) == outcome.traces[b]


@pytest.mark.parametrize("rank,world", [(0, 2), (1, 2), (3, 4), (7, 8)])
def test_rank_patching_matches_the_oracle(foundry, load, oracle, archives, rank, world):
    arch, _ = archives("moe-spmd")
    h = load(arch, rank=rank, world=world)
    want = expected_traces(oracle, arch, rank, world)
    for b in (1, 7, 16, 100, 255, 512):
        text = h.replay(b)
        assert text == want[b]
        assert "stub_" not in text
        assert "nccl_ring_allreduce" in text and "nvshmem_alltoall_ll" in text


def test_ranks_share_one_device_with_relocation(foundry, load, oracle, archives):
    """Several ranks on one GPU: only the first lands at the captured base; the
    others are relocated (K1) onto wherever the driver placed their region."""
    arch, _ = archives("moe-spmd")
    base = manifest(arch)["allocator"]["base"]
    handles = [load(arch, rank=r, world=4, relocate=True) for r in range(4)]
    bases = [h.region_base() for h in handles]
    assert len(set(bases)) == 4 and bases[0] == base
    for r, h in enumerate(handles):
        want = expected_traces(oracle, arch, r, 4, bases[r] - base)
        for b in (1, 64, 333):
            assert h.replay(b) == want[b]
        assert h.timings()["relocation_delta"] == bases[r] - base
    costs = [h.counters()["exec.instantiate_calls"] for h in handles]
    assert len(set(costs)) == 1


def test_shifted_base_without_relocation_fails_at_replay(foundry, load, archives):
    arch, _ = archives("micro")
    h = load(arch, base_shift_granules=1)
    with pytest.raises(foundry.FoundryError, match="unmapped-address"):
        h.replay(1)


def test_shifted_base_with_relocation_replays(foundry, load, oracle, archives):
    arch, _ = archives("micro")
    h = load(arch, base_shift_granules=1, relocate=True)
    want = expected_traces(oracle, arch, 0, 1, 0x10000)
    for b in h.batches():
        assert h.replay(b) == want[b]


def test_skip_restore_is_an_unresolved_kernel(foundry, load, archives):
    arch, _ = archives("micro")
    with pytest.raises(foundry.FoundryError, match="unresolved-kernel: template construction"):
        load(arch, skip_binary_restore=True)


def test_extra_prewindow_alloc_is_a_layout_divergence(foundry, load, archives):
    arch, _ = archives("micro")
    with pytest.raises(foundry.FoundryError, match="layout-divergence: foreground init"):
        load(arch, extra_prewindow_alloc=True)


def test_skip_device_init_fails_on_comm_nodes(foundry, load, archives):
    arch, _ = archives("moe-spmd")
    h = load(arch, skip_device_init=True)
    with pytest.raises(foundry.FoundryError, match="device-state-uninitialized"):
        h.replay(1)


def test_corrupt_graphs_bin_is_named(foundry, load, archives, tmp_path):
    arch, _ = archives("micro")
    bad = tmp_path / "bad"
    shutil.copytree(arch, bad)
    data = bytearray((bad / "graphs.bin").read_bytes())
    data[len(data) // 2] ^= 1
    (bad / "graphs.bin").write_bytes(bytes(data))
    with pytest.raises(foundry.FoundryError, match="archive-corruption: archive integrity: integrity check failed for graphs.bin"):
        load(str(bad))


def test_prepared_params_equal_the_oracle_records(foundry, load, oracle, archives):
    import fndg as F
    arch, _ = archives("moe-spmd")
    h = load(arch, rank=2, world=4)
    container, _ = oracle.materialize_archive(arch, 2, 4)
    recs = F.records(container)
    for b in (1, 2, 31, 32, 511, 512):
        assert h.prepared_record(b) == recs[b]


def test_serve_touches_only_differing_nodes(foundry, load, archives):
    arch, _ = archives("micro")
    h = load(arch)
    assert h.serve(1) == 0          # representative already applied
    touched = h.serve(2)
    assert touched > 0
    assert h.serve(2) == 0          # serving the applied member is free
    c = h.counters()
    assert c["exec.update_calls"] == 1
    assert c["exec.update_nodes_touched"] == touched


@pytest.mark.parametrize("name,batch", [("micro", 5), ("moe-spmd", 200), ("llama3-8b", 35)])
def test_materialized_graph_reproduces_a_fresh_capture(foundry, load, archives, name, batch):
    arch, _ = archives(name)
    h = load(arch)
    ok, report = h.fresh_capture_check(batch)
    assert ok, report


def test_reference_written_archive_loads(foundry, load, oracle, archives, tmp_path):
    """An archive without the B200 artefacts (as the reference writes it) is
    packed in memory at LOAD and replays identically."""
    arch, _ = archives("micro", b200=False)
    h = load(arch)
    want = expected_traces(oracle, arch)
    for b in h.batches():
        assert h.replay(b) == want[b]


def test_naive_rebuild_costs_more_construction(foundry, load, archives):
    arch, outcome = archives("micro")
    h = load(arch)
    naive = h.naive_rebuild_all()
    c = h.counters()
    templated = c["graph.add_node_calls"] + c["graph.add_edge_calls"] + c["graph.set_attr_calls"] + c["exec.instantiate_calls"]
    assert naive / templated >= 8 / 3 - 0.01


def _without_node_attrs(g):
    for n in g.nodes:
        n.attrs = b""
    return g


@pytest.mark.parametrize("name,rank,world,relocate", [
    ("micro", 0, 1, False), ("llama3-8b", 0, 1, False), ("moe-spmd", 1, 4, False), ("moe-spmd", 2, 4, True),
])
def test_gpu_capture_extracts_the_oracle_graph(foundry, load, oracle, archives, name, rank, world, relocate):
    """GPU-side SAVE: the member's work is stream-captured on
    the device with the template's dependencies, and the driver's graph is
    extracted back (cuGraphGetNodes/GetEdges, cuGraphKernelNodeGetParams +
    cuFuncGetParamInfo flattening). The FNDG record equals the oracle's
    materialized member byte for byte, except the per-node launch attributes
    the hardware cannot carry (reference cluster dims that do not divide the
    grid): those are compared where they were applied."""
    arch, _ = archives(name)
    base = manifest(arch)["allocator"]["base"]
    if relocate:  # a second handle holds the captured base: this one is relocated
        load(arch, rank=0, world=world)
    h = load(arch, rank=rank, world=world, relocate=relocate)
    delta = h.region_base() - base
    assert (delta != 0) == relocate
    container, _ = oracle.materialize_archive(arch, rank, world, delta)
    want = {g.label: g for g in fndg.graphs(container)}
    for b in h.batches()[:: max(1, len(h.batches()) // 12)]:
        got = fndg.decode_record(h.capture_graph(b))
        ref = want[b]
        assert got.label == b and len(got.nodes) == len(ref.nodes)
        assert got.edges == ref.edges
        for gn, rn in zip(got.nodes, ref.nodes):
            assert (gn.type, gn.grid, gn.block, gn.shmem, gn.hash, gn.name, gn.fattrs, gn.args, gn.mem) == \
                   (rn.type, rn.grid, rn.block, rn.shmem, rn.hash, rn.name, rn.fattrs, rn.args, rn.mem), \
                   "batch %d node %d" % (b, gn.id)
            if gn.type == 0 and rn.attrs[12:16] != b"\0\0\0\0":
                # an explicitly applied scheduling policy (i32 after the 3 x u32
                # cluster dims) reads back; an unset one reads back as the
                # driver's effective default, which the model cannot tell apart
                assert gn.attrs[12:16] == rn.attrs[12:16], "batch %d node %d policy" % (b, gn.id)


@pytest.mark.parametrize("name,rank,world", [("llama3-8b", 0, 1), ("moe-spmd", 3, 4)])
def test_shared_execs_serve_every_batch_like_the_oracle(foundry, load, oracle, archives, name, rank, world):
    """LoadOptions.share_execs: templates of one graph shape share an exec, so
    LOAD instantiates once per shape; serving still reproduces every member
    (switching the exec between templates in both directions)."""
    arch, outcome = archives(name)
    h = load(arch, rank=rank, world=world, share_execs=True)
    c = h.counters()
    assert 1 <= c["exec.instantiate_calls"] < outcome.template_count
    want = expected_traces(oracle, arch, rank, world)
    order = h.batches() + h.batches()[::-1]  # crosses every template boundary both ways
    for b in order:
        assert h.replay(b) == want[b], "batch %d" % b
    ok, report = h.fresh_capture_check(h.batches()[-1])
    assert ok, report


def test_exec_update_with_a_mismatched_donor_is_a_topology_mismatch(foundry, load, oracle, archives):
    """Acceptance criterion 7, last case (acceptance.cpp:304-371): updating an
    exec from a graph of another topology fails with topology-mismatch and
    leaves serving intact; a same-topology donor is applied."""
    arch, _ = archives("moe-spmd")
    h = load(arch)
    container, _ = oracle.materialize_archive(arch, 0, 1, 0)
    recs = fndg.records(container)
    want = expected_traces(oracle, arch)
    first, last = h.batches()[0], h.batches()[-1]
    with pytest.raises(foundry.FoundryError, match="topology-mismatch"):
        h.exec_update(first, recs[last])        # batch 1 and 512 are different templates
    h.exec_update(last, recs[last - 1])         # same template: applied node by node
    assert h.replay(last) == want[last]         # serving re-applies the member
    assert h.replay(first) == want[first]


@pytest.mark.parametrize("name,rank,world,relocate", [("llama3-8b", 0, 1, False), ("moe-spmd", 3, 4, True)])
def test_device_updates_serve_every_batch_like_the_oracle(foundry, load, oracle, archives, name, rank, world,
                                                          relocate):
    """LoadOptions.device_updates: kernel nodes are device-updatable and serve()
    applies each member from the GPU (cudaGraphKernelNodeSetParam/SetGridDim
    from the HBM member images); memcpy/memset nodes from the host. Every
    replay's on-device trace records must equal the oracle's, in both sweep
    directions (every template switch and member change)."""
    arch, _ = archives(name)
    base = manifest(arch)["allocator"]["base"]
    if relocate:
        load(arch, rank=0, world=world)
    h = load(arch, rank=rank, world=world, relocate=relocate, device_updates=True)
    want = expected_traces(oracle, arch, rank, world, h.region_base() - base)
    for b in h.batches() + h.batches()[::-1]:
        assert h.replay(b) == want[b], "batch %d" % b
    ok, report = h.fresh_capture_check(h.batches()[len(h.batches()) // 2])
    assert ok, report
    with pytest.raises(foundry.FoundryError, match="exclude each other"):
        load(arch, share_execs=True, device_updates=True)


def test_headline_graph_set_replay_verified(foundry, load, oracle, archives):
    """BASELINE config 5 at full size (qwen3-235b-a22b~ TP8, 512 graphs x 1036
    nodes): LOAD rank 5 of 8 through the public API, replay batches across
    every template against the oracle, and one fresh-capture equivalence."""
    arch, outcome = archives("qwen3-235b-a22b")
    h = load(arch, rank=5, world=8)
    assert h.counters()["exec.instantiate_calls"] == outcome.template_count == 12
    want = expected_traces(oracle, arch, 5, 8)
    for b in (1, 15, 16, 31, 47, 63, 95, 127, 191, 255, 319, 383, 447, 511, 512):
        assert h.replay(b) == want[b], "batch %d" % b
    ok, report = h.fresh_capture_check(300)
    assert ok, report


@pytest.mark.parametrize("name", ["micro", "dense-small", "moe-spmd"])
def test_layout_determinism_with_and_without_preallocation(foundry, load, archives, name):
    """Acceptance criterion 2 (acceptance.cpp:143-161): LOAD reproduces SAVE's
    allocation addresses, with the one-shot preallocation and without it."""
    arch, outcome = archives(name)
    assert outcome.allocation_records
    for pre in (True, False):
        h = load(arch, preallocate=pre)
        assert h.allocation_records() == outcome.allocation_records, "preallocate=%s" % pre
        h.close()


def test_construction_reduction_on_dense_small(foundry, load, archives):
    """Acceptance criterion 4 (acceptance.cpp:182-220) on real graphs: dense-small
    has 20 templates; templated construction (graph mutation + instantiate)
    times 512 stays within the naive rebuild times K+1, and with the
    per-member updates of serving every batch the ratio is <= 0.10."""
    arch, outcome = archives("dense-small")
    assert outcome.template_count == 20
    h = load(arch)
    for b in h.batches():
        h.serve(b)
    c = h.counters()
    templated = (c["graph.add_node_calls"] + c["graph.add_edge_calls"] + c["graph.set_attr_calls"]
                 + c["exec.instantiate_calls"])
    updates = c["exec.update_calls"]
    naive = h.naive_rebuild_all()
    assert templated * 512 <= naive * (outcome.template_count + 1)
    assert (templated + updates) / naive <= 0.10


@pytest.mark.parametrize("name", ["micro", "dense-small"])
def test_replay_equivalence_at_world_four(foundry, load, oracle, archives, name):
    """Acceptance criterion 1 (acceptance.cpp:108-141) at W=4: every batch of
    rank 3 replays exactly the oracle's trace."""
    arch, _ = archives(name)
    h = load(arch, rank=3, world=4)
    want = expected_traces(oracle, arch, 3, 4)
    for b in h.batches():
        assert h.replay(b) == want[b], "batch %d" % b


@pytest.mark.parametrize("fail", [False, True])
def test_device_updates_random_serve_order(foundry, load, oracle, archives, fail):
    """Asynchronous device serves in a random order, interleaved with serves
    that are not replayed (queued updates overwritten by later ones) and
    with repeated batches: every replay still matches the oracle. With
    fail=True every device update reports failure (FaultInjection
    fail_device_serve): replay() finds the error flags at its synchronization
    point, re-applies the failed members on the host and launches again."""
    import random
    arch, _ = archives("moe-spmd")
    h = load(arch, rank=2, world=8, device_updates=True, fail_device_serve=fail)
    want = expected_traces(oracle, arch, 2, 8)
    rng = random.Random(11)
    bs = h.batches()
    for i in range(150):
        b = rng.choice(bs)
        for _ in range(rng.randrange(3)):
            h.serve(rng.choice(bs))  # queued, superseded
        if i % 3 == 0:
            h.serve(b)
            h.serve(b)               # no-op: already applied
        assert h.replay(b) == want[b], "step %d batch %d" % (i, b)


@pytest.mark.parametrize("share", [False, True])
def test_restored_shared_memory_limits_allow_large_launches(foundry, load, oracle, archives, tmp_path, share):
    """Function attributes recorded at capture are restored at LOAD: every
    kernel node launches with as much dynamic shared memory as its recorded
    MAX_DYNAMIC_SHARED_SIZE_BYTES allows (> 48 KiB), which the device accepts
    only if the limit was applied to the function the graph launches."""
    import tier_s
    src, _ = archives("moe-spmd")
    arch = tier_s.make_big_smem(src, str(tmp_path / "big"), oracle.crc64)
    foundry._foundry._pack_store(arch)
    h = load(arch, rank=1, world=4, share_execs=share)
    want = expected_traces(oracle, arch, 1, 4)
    for b in h.batches()[::17] + [h.batches()[-1]]:
        assert h.replay(b) == want[b], "batch %d" % b
    import re
    assert max(int(x) for x in re.findall(r"shmem=(\d+)", want[h.batches()[-1]])) > 48 * 1024
