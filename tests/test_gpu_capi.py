"""GPU parity through the C-ABI (include/foundry_b200.h) — the boundary a
foreign host binds. Every materialized member-image arena is
decoded back to FNDG records and compared byte for byte with the C oracle's
materialization of the same archive (parse_graph_at + relocation + rank
patch), which test_oracle.py pins to the reference.
"""
from __future__ import annotations

import ctypes
import json
import os
import shutil
import socket
import subprocess
import sys

import pytest

from conftest import ROOT, manifest

pytestmark = pytest.mark.gpu

ERR_INVALID_ARGUMENT = 1
ERR_ARCHIVE_CORRUPTION = 8

# deltas {0, one granule, 0x7000.. -> 0x7100.., a SplitMix64 draw}
DELTAS = [0, 0x10000, 0x10000000000, 0x5A3F2B0000]


@pytest.fixture(scope="module")
def api(foundry):
    from paper_2604_06664_b200 import capi
    return capi.CApi()


@pytest.fixture(scope="module")
def dev(api):
    d = api.device_open(0)
    yield d
    api.lib.fdy_device_close(d)


def decode(foundry, arch, arena: bytes) -> bytes:
    return foundry._foundry._decode_member_images(arch, arena)


@pytest.mark.parametrize("name,rank,world,delta", [
    ("micro", 0, 1, 0),
    ("llama3-8b", 0, 1, DELTAS[1]),
    ("moe-spmd", 3, 8, DELTAS[2]),
    ("moe-spmd", 7, 8, DELTAS[3]),
])
def test_materialize_equals_the_oracle(foundry, oracle, archives, api, dev, name, rank, world, delta):
    arch, _ = archives(name)
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    base = manifest(arch)["allocator"]["base"]
    store = api.store_upload(dev, blob)
    try:
        members, ms = api.materialize(dev, store, rank, world, base + delta if delta else 0)
        assert ms > 0
        got = decode(foundry, arch, api.members_download(members))
        api.lib.fdy_members_free(members)
    finally:
        api.lib.fdy_store_free(store)
    want, _ = oracle.materialize_archive(arch, rank, world, delta)
    assert got == want


def test_materialize_into_reuses_the_arena(foundry, oracle, archives, api, dev):
    """fdy_materialize_into overwrites every byte: ranks alternate in one arena."""
    arch, _ = archives("moe-spmd")
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    base = manifest(arch)["allocator"]["base"]
    store = api.store_upload(dev, blob)
    members, _ = api.materialize(dev, store, 0, 4)
    try:
        for rank, delta in ((1, DELTAS[1]), (2, 0), (3, DELTAS[3])):
            api.materialize(dev, store, rank, 4, base + delta if delta else 0, members)
            want, _ = oracle.materialize_archive(arch, rank, 4, delta)
            assert decode(foundry, arch, api.members_download(members)) == want, (rank, hex(delta))
    finally:
        api.lib.fdy_members_free(members)
        api.lib.fdy_store_free(store)


@pytest.mark.parametrize("name,rank,world,delta", [("micro", 0, 1, 0), ("moe-spmd", 3, 4, DELTAS[3])])
def test_member_pass_writes_every_arena_byte(archives, api, dev, name, rank, world, delta):
    """The member pass writes the arena with TMA bulk stores, which
    compute-sanitizer initcheck does not model (tools/initcheck.sh flags every
    D2H of the arena). Raw bytes, padding included: an arena filled with a
    pattern (fdy_members_write_probe) and materialized again must equal the
    first materialization byte for byte."""
    arch, _ = archives(name)
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    base = manifest(arch)["allocator"]["base"]
    store = api.store_upload(dev, blob)
    members, _ = api.materialize(dev, store, rank, world, base + delta if delta else 0)
    try:
        first = api.members_download(members)
        ms = ctypes.c_float()
        api.check(api.lib.fdy_members_write_probe(members, ctypes.byref(ms)))
        assert api.members_download(members) != first  # the pattern landed
        api.materialize(dev, store, rank, world, base + delta if delta else 0, members)
        assert api.members_download(members) == first
    finally:
        api.lib.fdy_members_free(members)
        api.lib.fdy_store_free(store)


@pytest.mark.parametrize("name,seed", [("micro", 0), ("moe-spmd", 1)])
def test_forged_store_is_rejected_or_contained(archives, tmp_path, name, seed):
    """templates.fdt with random byte flips and a matching manifest digest
    (tests/store_fuzz_worker.py): fdy_prepare_archive and LOAD + replay either
    succeed or raise a non-CUDA FoundryError; the store's table validation
    (StoreView), the member pass's lane / chunk clamps and the image
    descriptor checks keep a forged store off the device's out-of-bounds
    paths. Run in a subprocess so a device fault could not poison this one."""
    arch, _ = archives(name)
    n = os.environ.get("FOUNDRY_FUZZ_N", "24")
    seed += 7919 * int(os.environ.get("FOUNDRY_FUZZ_ROUND", "0"))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "store_fuzz_worker.py"), arch,
                          str(tmp_path), str(seed), n], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["ok"] + res["rejected"] == int(n) and res["rejected"] > 0, res


def test_rank_outside_world_is_invalid_argument(archives, api, dev):
    from paper_2604_06664_b200.capi import CApiError
    arch, _ = archives("micro")
    store = api.store_upload(dev, open(os.path.join(arch, "templates.fdt"), "rb").read())
    try:
        with pytest.raises(CApiError, match="outside world size") as e:
            api.materialize(dev, store, 4, 4)
        assert e.value.code == ERR_INVALID_ARGUMENT
    finally:
        api.lib.fdy_store_free(store)


def test_store_fanout_to_the_same_device(foundry, oracle, archives, api, dev):
    """fdy_store_fanout (GPU -> GPU copy); on one GPU the copy is device-local."""
    arch, _ = archives("moe-spmd")
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    src = api.store_upload(dev, blob)
    out = ctypes.c_void_p()
    api.check(api.lib.fdy_store_fanout(src, dev, ctypes.byref(out)))
    api.lib.fdy_store_free(src)  # the copy must stand alone
    try:
        members, _ = api.materialize(dev, out, 5, 8)
        got = decode(foundry, arch, api.members_download(members))
        api.lib.fdy_members_free(members)
    finally:
        api.lib.fdy_store_free(out)
    want, _ = oracle.materialize_archive(arch, 5, 8, 0)
    assert got == want


@pytest.mark.parametrize("b200", [True, False])
@pytest.mark.parametrize("rank,world,delta", [(0, 1, 0), (6, 8, DELTAS[2])])
def test_prepare_archive_equals_the_oracle(foundry, oracle, archives, api, dev, b200, rank, world, delta):
    """fdy_prepare_archive: files -> GPU integrity -> fused kernel -> host memory,
    for a B200 archive (store on disk) and a reference-written one (packed on the fly)."""
    from paper_2604_06664_b200 import capi
    arch, _ = archives("moe-spmd", b200=b200)
    base = manifest(arch)["allocator"]["base"]
    size = capi.store_header(open(os.path.join(archives("moe-spmd")[0], "templates.fdt"), "rb").read())[
        "members_image_bytes"]  # same spec, same member images
    host = api.host_alloc(dev, size)
    try:
        t = api.prepare_archive(dev, arch, rank, world, base + delta if delta else 0, 4, host, size)
        arena = ctypes.string_at(host, t["member_bytes"])
    finally:
        api.lib.fdy_host_free(host)
    assert t["graphs"] == 512 and t["d2h_bytes"] == t["member_bytes"]
    want, _ = oracle.materialize_archive(arch, rank, world, delta)
    # decoded with the B200 archive's store: packing is deterministic, so the
    # store packed on the fly from the plain archive has the same layout
    assert decode(foundry, archives("moe-spmd")[0], arena) == want


@pytest.mark.parametrize("victim", ["graphs.bin", "templates.fdt", "catalog.bin"])
def test_prepare_archive_names_the_corrupt_file(archives, api, dev, tmp_path, victim):
    from paper_2604_06664_b200.capi import CApiError
    arch, _ = archives("micro")
    bad = tmp_path / "bad"
    shutil.copytree(arch, bad)
    data = bytearray((bad / victim).read_bytes())
    data[len(data) // 3] ^= 0x40
    (bad / victim).write_bytes(bytes(data))
    host = api.host_alloc(dev, 64 << 20)
    try:
        with pytest.raises(CApiError, match="archive integrity: integrity check failed for " + victim) as e:
            api.prepare_archive(dev, str(bad), 0, 1, 0, 4, host, 64 << 20)
        assert e.value.code == ERR_ARCHIVE_CORRUPTION
    finally:
        api.lib.fdy_host_free(host)


def test_prepare_archive_reports_the_first_corrupt_file_in_manifest_order(archives, api, dev, tmp_path):
    """Two corrupt files: the one earlier in manifest order is named (as the
    reference's verify_archive_integrity walk would), even though the store
    is verified first."""
    from paper_2604_06664_b200.capi import CApiError
    arch, _ = archives("micro")
    bad = tmp_path / "bad2"
    shutil.copytree(arch, bad)
    for victim in ("graphs.bin", "templates.fdt"):
        data = bytearray((bad / victim).read_bytes())
        data[7] ^= 1
        (bad / victim).write_bytes(bytes(data))
    host = api.host_alloc(dev, 64 << 20)
    try:
        with pytest.raises(CApiError, match="integrity check failed for graphs.bin"):
            api.prepare_archive(dev, str(bad), 0, 1, 0, 4, host, 64 << 20)
    finally:
        api.lib.fdy_host_free(host)


@pytest.mark.parametrize("sizes", [
    [0], [1], [15, 16, 17], [65535, 65536, 65537], [3 * 65536 + 5, 0, 999_999], [8 << 20],
])
def test_crc64_segments_match_the_oracle(oracle, api, dev, sizes):
    import random
    rng = random.Random(sum(sizes) + len(sizes))
    parts, ranges, off = [], [], 0
    for n in sizes:
        data = bytes(rng.getrandbits(8) for _ in range(min(n, 4096))) * (n // 4096 + 1)
        data = data[:n]
        parts.append(data + b"\0" * ((-len(data)) % 16))  # segments start 16-byte aligned
        ranges.append((off, n))
        off += len(parts[-1])
    digests, _ = api.crc64(dev, b"".join(parts), ranges)
    assert digests == [oracle.crc64(p[:n]) for p, (_, n) in zip(parts, ranges)]


def test_crc64_known_answer(api, dev):
    """crc64("123456789") == 0x995DC9BBDF1939FA (test_hash.cpp:13-16)."""
    digests, _ = api.crc64(dev, b"123456789", [(0, 9)])
    assert digests == [0x995DC9BBDF1939FA]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_ipc_fanout_between_two_processes(foundry, oracle, archives, tmp_path):
    """The N>1 exchange step on one GPU: rank 0 uploads + exports the store
    (CUDA IPC), rank 1 imports it GPU -> GPU; each materializes its own TP
    rank and must equal the oracle's graph set for that rank."""
    arch, _ = archives("moe-spmd")
    port = _free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                   WORLD_SIZE="2", LOCAL_RANK=str(rank))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "ipc_worker.py"), arch,
                                       str(tmp_path)], env=env))
    for p in procs:
        assert p.wait(timeout=600) == 0
    for rank in range(2):
        got = (tmp_path / ("rank%d.fndg" % rank)).read_bytes()
        want, _ = oracle.materialize_archive(arch, 2 + rank, 8, 0x10000 * (rank + 1))
        assert got == want, rank


def test_chain_fanout_between_three_processes(foundry, oracle, archives, tmp_path):
    """SURVEY §8(e) option ii across processes: rank 0 seeds a pipelined chain
    from host memory, rank 1 pulls every chunk from rank 0 and rank 2 from
    rank 1 as each lands (GPU-polled progress words over CUDA IPC); each rank
    materializes its own TP rank from its copy and must equal the oracle."""
    arch, _ = archives("moe-spmd")
    port = _free_port()
    procs = []
    for rank in range(3):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                   WORLD_SIZE="3", LOCAL_RANK=str(rank))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "ipc_worker.py"), arch,
                                       str(tmp_path), "chain"], env=env))
    for p in procs:
        assert p.wait(timeout=600) == 0
    for rank in range(3):
        got = (tmp_path / ("rank%d.fndg" % rank)).read_bytes()
        want, _ = oracle.materialize_archive(arch, 2 + rank, 8, 0x10000 * (rank + 1))
        assert got == want, rank


def test_chain_link_times_out_on_a_silent_predecessor(tmp_path):
    """A chain link whose predecessor never publishes gives up after the
    timeout (the GPU's wait kernel stops polling) and fdy_chain_finish raises,
    instead of hanging its GPU's stream; the link after it gives up as well
    (a link that gave up forwards nothing)."""
    port = _free_port()
    procs = []
    for rank in range(3):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                   WORLD_SIZE="3", LOCAL_RANK=str(rank))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "chain_timeout_worker.py")],
                                      env=env))
    assert [p.wait(timeout=300) for p in procs] == [0, 0, 0]


@pytest.mark.parametrize("chunk", [0, 4096 + 16])
def test_chain_fanout_in_one_process(foundry, oracle, archives, api, dev, chunk):
    """fdy_store_fanout_chain through three device handles (one GPU here, so
    each hop is a device-to-device copy on its own stream, ordered by the
    per-chunk events exactly as across GPUs); every link's store materializes
    like the oracle. chunk = 4112 bytes: many chunks, ragged last one."""
    arch, _ = archives("moe-spmd")
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    devs = [api.device_open(0) for _ in range(3)]
    src = api.store_upload(dev, blob)
    outs = api.store_fanout_chain(src, devs, chunk)
    base = manifest(arch)["allocator"]["base"]
    try:
        for i, (d, st) in enumerate(zip(devs, outs)):
            members, _ = api.materialize(d, st, i + 1, 4, base)
            try:
                got = decode(foundry, arch, api.members_download(members))
            finally:
                api.lib.fdy_members_free(members)
            want, _ = oracle.materialize_archive(arch, i + 1, 4, 0)
            assert got == want, i
    finally:
        for st in outs:
            api.lib.fdy_store_free(st)
        api.lib.fdy_store_free(src)
        for d in devs:
            api.lib.fdy_device_close(d)


def test_session_layer_load_replay_and_capture(foundry, oracle, archives, api):
    """The reference's LOAD surface through the C-ABI (fdy_load ->
    fdy_serving_replay / fdy_serving_capture_graph): traces equal the oracle's,
    and the GPU-captured graph record equals the oracle's member record except
    for node launch attributes (test_gpu_pipeline.py explains which)."""
    import fndg

    arch, _ = archives("moe-spmd")
    container, _ = oracle.materialize_archive(arch, 5, 8, 0)
    graphs = {g.label: g for g in fndg.graphs(container)}
    hidden = fndg.hidden_map(arch)
    h = api.load(arch, rank=5, world=8)
    try:
        for b in (1, 2, 9, 100, 512):
            assert api.serving_replay(h, b) == fndg.trace_text(graphs[b], hidden, oracle.crc64)
            got = fndg.decode_record(api.serving_capture_graph(h, b))
            ref = graphs[b]
            assert got.edges == ref.edges
            assert [(n.type, n.grid, n.block, n.shmem, n.name, n.args, n.mem) for n in got.nodes] == \
                   [(n.type, n.grid, n.block, n.shmem, n.name, n.args, n.mem) for n in ref.nodes]
    finally:
        api.lib.fdy_serving_close(h)


# BASELINE.json configs at their full tier-R sizes: the
# spec, then the (rank, world, delta) cases each config is quoted on.
FULL_CONFIGS = [
    ("llama3-8b", [(0, 1, 0x10000)]),                                   # config 1, TP=1
    ("qwen3-8b", [(0, 1, 0x10000000000)]),                              # config 2, TP=1
    ("qwen3-30b-a3b", [(0, 1, 0), (1, 2, 0x10000)]),                    # config 3, 1 and 2 GPUs
    ("llama3-70b", [(3, 4, 0x10000), (7, 8, DELTAS[3])]),              # config 4, TP4 / TP8
    ("qwen3-235b-a22b", [(r, 8, [0x10000, DELTAS[2], DELTAS[3], 0][r % 4]) for r in range(8)]),  # config 5: all 8 TP ranks
]


@pytest.mark.parametrize("name,cases", FULL_CONFIGS, ids=[c[0] for c in FULL_CONFIGS])
def test_baseline_configs_full_size_bit_exact(foundry, oracle, api, dev, tmp_path, name, cases):
    """Every BASELINE config at full size through the C-ABI: the GPU-CRC'd
    archive files equal their manifest digests, and every member graph of
    every (rank, world, delta) case equals the oracle byte for byte."""
    from conftest import spec_path

    arch = str(tmp_path / name)
    foundry.save(foundry.workload_from_text(open(spec_path(name)).read()), arch, b200_artifacts=False)
    foundry._foundry._pack_store(arch)
    m = manifest(arch)
    files = sorted(f for f in m["files"] if f != "templates.fdt") + ["templates.fdt"]
    parts, ranges, off = [], [], 0
    for f in files:
        d = open(os.path.join(arch, f), "rb").read()
        parts.append(d + b"\0" * ((-len(d)) % 256))
        ranges.append((off, len(d)))
        off += len(parts[-1])
    digests, _ = api.crc64(dev, b"".join(parts), ranges)
    want_digests = dict(m["files"])
    for f, dg in zip(files, digests):
        if f in want_digests:
            assert dg == want_digests[f], f
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    base = m["allocator"]["base"]
    store = api.store_upload(dev, blob)
    try:
        for rank, world, delta in cases:
            members, _ = api.materialize(dev, store, rank, world, base + delta if delta else 0)
            try:
                got = decode(foundry, arch, api.members_download(members))
            finally:
                api.lib.fdy_members_free(members)
            want, _ = oracle.materialize_archive(arch, rank, world, delta)
            assert got == want, (name, rank, world, hex(delta))
    finally:
        api.lib.fdy_store_free(store)


@pytest.mark.parametrize("name,rank,world,delta", [
    ("moe-spmd", 0, 1, 0), ("moe-spmd", 3, 8, 0x10000), ("moe-spmd", 5, 8, DELTAS[3]),
    ("qwen3-235b-a22b", 5, 8, 0x10000),  # the bench's tier-S arena (330 MB of member images)
])
def test_tier_s_graphs_on_the_gpu(foundry, oracle, archives, api, dev, tmp_path, name, rank, world, delta):
    """Tier-S fixtures (tests/tier_s.py: 1720-byte argument blocks, unaligned
    pointers, ragged sizes, member-varying grids) through the fused kernel."""
    import tier_s
    src, _ = archives(name)
    arch = tier_s.make_tier_s(src, str(tmp_path / "s"), oracle.crc64)
    foundry._foundry._pack_store(arch)
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    base = manifest(arch)["allocator"]["base"]
    store = api.store_upload(dev, blob)
    try:
        members, _ = api.materialize(dev, store, rank, world, base + delta if delta else 0)
        try:
            got = decode(foundry, arch, api.members_download(members))
        finally:
            api.lib.fdy_members_free(members)
    finally:
        api.lib.fdy_store_free(store)
    want, _ = oracle.materialize_archive(arch, rank, world, delta)
    assert got == want
