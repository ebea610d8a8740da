"""K3 per-rank communication state on the GPU (north_star kernel 3: comm
handles and peer buffer addresses, beyond rank/world ids): the archive's
comm slots (comm_slots.bin, written by the stub layer) become FDT_ROP_VALUE
ops that the fused kernel fills from each rank's value table.

Parity: the C oracle applies the same slot rule after apply_rank_patches, and
test_store.py pins that rule against the reference's own PrepareFn output
(identical except at exactly the slot bytes)."""
from __future__ import annotations

import ctypes
import os
import shutil

import pytest

import comm_slots
import fndg
from conftest import manifest

pytestmark = pytest.mark.gpu

DELTAS = [0, 0x10000, 0x10000000000, 0x5A3F2B0000]


@pytest.fixture(autouse=True)
def _release_handles():
    import gc
    yield
    gc.collect()


@pytest.fixture(scope="module")
def api(foundry):
    from paper_2604_06664_b200 import capi
    return capi.CApi()


@pytest.fixture(scope="module")
def dev(api):
    d = api.device_open(0)
    yield d
    api.lib.fdy_device_close(d)


def slotted(foundry, archives, tmp_path, table_fn, name="moe-spmd", b200=True):
    arch, _ = archives(name, b200=b200)
    copy = str(tmp_path / (name + ("-slots" if b200 else "-plain-slots")))
    shutil.copytree(arch, copy)
    foundry.write_comm_slots(copy, comm_slots.N_VALUES, table_fn(copy))
    return copy


def test_eight_ranks_with_distinct_comm_state(foundry, oracle, archives, api, dev, tmp_path):
    """All 8 ranks of W=8 from ONE store upload, each with its own value table
    (comm handle + peer buffers) and a relocation delta: every member graph
    equals the oracle byte for byte (writes straddling chunks, 1/4/8-byte
    widths, slots over the rank/world bytes)."""
    arch = slotted(foundry, archives, tmp_path, comm_slots.stress_table)
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    base = manifest(arch)["allocator"]["base"]
    store = api.store_upload(dev, blob)
    members = None
    seen = set()
    try:
        for rank in range(8):
            delta = DELTAS[rank % 4]
            vals = comm_slots.rank_values(rank)
            members, _ = api.materialize(dev, store, rank, 8, base + delta if delta else 0, members, values=vals)
            got = foundry._foundry._decode_member_images(arch, api.members_download(members))
            want, _ = oracle.materialize_archive(arch, rank, 8, delta, values=vals)
            assert got == want, rank
            seen.add(got)
        assert len(seen) == 8
        # too few values for the archive's slots: invalid-argument, nothing launched
        from paper_2604_06664_b200.capi import CApiError
        with pytest.raises(CApiError, match="comm slots read 6 per-rank values, 2 given"):
            api.materialize(dev, store, 0, 8, 0, members, values=comm_slots.rank_values(0)[:2])
    finally:
        if members is not None:
            api.lib.fdy_members_free(members)
        api.lib.fdy_store_free(store)


def test_prepare_archive_applies_the_value_table(foundry, oracle, archives, api, dev, tmp_path):
    """fdy_prepare_archive (files -> GPU integrity -> fused kernel -> host)
    takes the descriptor's value table too."""
    arch = slotted(foundry, archives, tmp_path, comm_slots.stress_table)
    from paper_2604_06664_b200 import capi
    h = capi.store_header(open(os.path.join(arch, "templates.fdt"), "rb").read())
    base = manifest(arch)["allocator"]["base"]
    n = h["members_image_bytes"]
    out = api.host_alloc(dev, n)
    try:
        vals = comm_slots.rank_values(6)
        api.prepare_archive(dev, arch, 6, 8, base + 0x10000, 4, out, n, values=vals)
        got = foundry._foundry._decode_member_images(arch, ctypes.string_at(out, n))
    finally:
        api.lib.fdy_host_free(out)
    want, _ = oracle.materialize_archive(arch, 6, 8, 0x10000, values=vals)
    assert got == want


@pytest.mark.parametrize("share,b200", [(False, True), (True, True), (False, False)])
def test_load_with_comm_values_replays_like_the_oracle(foundry, load, oracle, archives, tmp_path, share, b200):
    """LOAD with LoadOptions.comm_values: the deploy table puts a peer buffer
    (a mapped region address, so the device dereference succeeds) at buf@16 and
    a comm handle over payload@24; every replayed trace equals the oracle's.
    b200=False: the archive in the reference's layout plus comm_slots.bin, so
    the GPU packer turns the slots into value ops at LOAD."""
    arch = slotted(foundry, archives, tmp_path, comm_slots.deploy_table, b200=b200)
    base = manifest(arch)["allocator"]["base"]
    rank = 3
    vals = comm_slots.rank_values(rank, base)
    with pytest.raises(foundry.FoundryError, match="invalid-argument.*comm slots read 6"):
        load(arch, rank=rank, world=8)
    h = load(arch, rank=rank, world=8, comm_values=vals, share_execs=share)
    container, _ = oracle.materialize_archive(arch, rank, 8, values=vals)
    hidden = fndg.hidden_map(arch)
    want = {g.label: fndg.trace_text(g, hidden, oracle.crc64) for g in fndg.graphs(container)}
    for b in h.batches()[::7] + [h.batches()[-1]]:
        assert h.replay(b) == want[b], "batch %d" % b
    assert ("%x" % vals[1]) in h.replay(1)  # a peer buffer address reached the trace
