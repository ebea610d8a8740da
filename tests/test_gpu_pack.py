"""GPU packer (kernels/pack.cu + host/device_pack.cpp).

A reference-written archive (graphs.bin + patch.bin, no templates.fdt) is
packed into the FNDT template store on the device at LOAD. The offline packer
(template_store.cpp pack_template_store) is itself pinned to the reference's
decode (parse_graph_at, graph_model.cpp:295-303) and, through the
materialization tests, to the oracle; so the GPU packer must produce the same
store byte for byte, raise the same errors for the same corruptions, and LOAD
such archives to graphs whose replays equal the oracle's.
"""
from __future__ import annotations

import json
import os
import shutil
import struct

import pytest

import fndg
from conftest import manifest
from test_gpu_pipeline import expected_traces

pytestmark = pytest.mark.gpu

SMALL = ["micro", "dense-small", "moe-spmd", "llama3-8b"]
FULL = ["qwen3-8b", "qwen3-30b-a3b", "llama3-70b", "qwen3-235b-a22b"]


def _first_difference(a: bytes, b: bytes) -> str:
    if len(a) != len(b):
        return "sizes %d != %d" % (len(a), len(b))
    for i in range(len(a)):
        if a[i] != b[i]:
            return "first difference at byte %d" % i
    return "equal"


def _same_store(foundry, arch):
    gpu, t = foundry._foundry._pack_store_bytes(arch, True)
    cpu, _ = foundry._foundry._pack_store_bytes(arch, False)
    assert gpu == cpu, _first_difference(gpu, cpu)
    assert t["retries"] == 0
    return t


@pytest.mark.parametrize("name", SMALL + FULL)
def test_gpu_pack_equals_the_offline_packer(foundry, archives, name):
    """Every BASELINE config (full size) and preset: the store built on the
    GPU equals the offline packer's, byte for byte."""
    arch, _ = archives(name, b200=False)
    t = _same_store(foundry, arch)
    assert t["kernel_keys"] > 0


def test_gpu_pack_tier_s_and_big_shared_memory(foundry, archives, oracle, tmp_path):
    """Model-shaped argument blocks (1720-byte GEMM blocks, ragged tails,
    member-varying grids) and recorded >48 KiB shared-memory limits."""
    import tier_s
    src, _ = archives("moe-spmd", b200=False)
    _same_store(foundry, tier_s.make_tier_s(src, str(tmp_path / "tier_s"), oracle.crc64))
    _same_store(foundry, tier_s.make_big_smem(src, str(tmp_path / "big"), oracle.crc64))


@pytest.mark.parametrize("table", ["stress", "deploy"])
def test_gpu_pack_comm_slots(foundry, archives, tmp_path, table):
    """Per-rank comm-state slots (comm_slots.bin) become the same value ops."""
    import comm_slots
    src, _ = archives("moe-spmd", b200=False)
    arch = str(tmp_path / "slots")
    shutil.copytree(src, arch)
    fn = comm_slots.stress_table if table == "stress" else comm_slots.deploy_table
    foundry.write_comm_slots(arch, comm_slots.N_VALUES, fn(arch))
    _same_store(foundry, arch)


@pytest.mark.parametrize("name,rank,world,relocate", [("micro", 0, 1, False), ("moe-spmd", 3, 8, True),
                                                      ("qwen3-30b-a3b", 1, 2, False)])
def test_load_of_a_reference_written_archive_packs_on_the_gpu(foundry, load, oracle, archives, name, rank, world,
                                                              relocate):
    """LOAD of an archive without templates.fdt: graphs.bin goes to HBM, the
    store is packed there (pack_ms), and every batch replays like the oracle."""
    arch, _ = archives(name, b200=False)
    base = manifest(arch)["allocator"]["base"]
    if relocate:
        load(arch, rank=0, world=world)  # holds the captured base: the next LOAD relocates
    h = load(arch, rank=rank, world=world, relocate=relocate)
    assert h.timings()["pack_ms"] > 0
    want = expected_traces(oracle, arch, rank, world, h.region_base() - base)
    for b in h.batches():
        assert h.replay(b) == want[b], "batch %d" % b


# ------------------------------------------------------------------ errors

def _rewrite(src: str, dst: str, crc64, edit) -> str:
    """Copy an archive, let `edit(graphs)` change its decoded graphs, and write
    graphs.bin back with fresh record checksums, locators and digest."""
    shutil.copytree(src, dst)
    m = json.load(open(os.path.join(dst, "manifest")))
    raw = open(os.path.join(dst, "graphs.bin"), "rb").read()
    (version,) = struct.unpack_from("<H", raw, 4)
    graphs = fndg.graphs(raw)
    edit(graphs)
    data, locs = fndg.write_container(graphs, version, crc64)
    _commit(dst, m, data, locs, crc64)
    return dst


def _commit(dst, m, data, locs, crc64):
    open(os.path.join(dst, "graphs.bin"), "wb").write(data)
    by_label = {l[0]: l for l in locs}
    for grp in m["grouping"]["groups"]:
        grp["locators"] = [list(by_label[l[0]]) for l in grp["locators"]]
    m["files"]["graphs.bin"] = crc64(data)
    m["files"].pop("templates.fdt", None)
    json.dump(m, open(os.path.join(dst, "manifest"), "w"))


def _non_representative(arch):
    m = manifest(arch)
    grp = max(m["grouping"]["groups"], key=lambda g: len(g["members"]))
    return [l[0] for l in grp["locators"] if l[0] != grp["representative"]][-1]


def _raw_edit(src, dst, crc64, label, fn):
    """Byte-level edit of one record (the decoder must reject it); the record
    checksum, locator and file digest are made consistent again."""
    shutil.copytree(src, dst)
    m = json.load(open(os.path.join(dst, "manifest")))
    raw = bytearray(open(os.path.join(dst, "graphs.bin"), "rb").read())
    locs = fndg.locators(bytes(raw))
    for i, (lab, off, length, _) in enumerate(locs):
        if lab == label:
            rec = bytearray(raw[off:off + length])
            fn(rec)
            raw[off:off + length] = rec
            struct.pack_into("<Q", raw, 10 + 28 * i + 20, crc64(bytes(rec)))
            locs[i] = (lab, off, length, crc64(bytes(rec)))
    _commit(dst, m, bytes(raw), locs, crc64)
    return dst


def _errors(foundry, load, arch):
    with pytest.raises(foundry.FoundryError) as gpu:
        foundry._foundry._pack_store_bytes(arch, True)
    with pytest.raises(foundry.FoundryError) as cpu:
        foundry._foundry._pack_store_bytes(arch, False)
    assert str(gpu.value) == str(cpu.value)
    with pytest.raises(foundry.FoundryError) as ld:
        load(arch, rank=1, world=2)
    assert "template construction" in str(ld.value)
    assert str(cpu.value).split(": ", 1)[1] in str(ld.value)
    return str(gpu.value)


def _kernel_node(graphs, label, pred=lambda n: True):
    g = next(g for g in graphs if g.label == label)
    return g, next(n for n in g.nodes if n.type == 0 and pred(n))


def test_errors_match_the_offline_packer(foundry, load, oracle, archives, tmp_path):
    """Corruptions of one member record (consistent checksums, so integrity
    passes): the GPU packer raises exactly the offline packer's error, and
    LOAD reports it under "template construction"."""
    src, _ = archives("moe-spmd", b200=False)
    crc = oracle.crc64
    victim = _non_representative(src)
    stubs = fndg.patch_nodes(open(os.path.join(src, "patch.bin"), "rb").read())

    def drop_edge(gs):
        next(g for g in gs if g.label == victim).edges.pop()

    def empty_args(gs):
        _kernel_node(gs, victim)[1].args = b""

    def zero_grid(gs):
        n = _kernel_node(gs, victim)[1]
        n.grid = (0, n.grid[1], n.grid[2])

    def backwards_edge(gs):
        g = next(g for g in gs if g.label == victim)
        f, t = g.edges[0]
        g.edges[0] = (t, f)

    def wrong_stub(gs):
        g = next(g for g in gs if g.label == victim)
        g.nodes[stubs[victim][0]].hash ^= 1

    cases = {
        "topology": (drop_edge, "topology-mismatch"),
        "empty args": (empty_args, "empty argument buffer"),
        "launch dims": (zero_grid, "launch dims must be >= 1"),
        "edge order": (backwards_edge, "edge must go from an earlier node"),
        "stub": (wrong_stub, "is not the recorded stub"),
    }
    for case, (edit, want) in cases.items():
        arch = _rewrite(src, str(tmp_path / case.replace(" ", "_")), crc, edit)
        assert want in _errors(foundry, load, arch), case

    def bad_tag(rec):
        rec[12] = 7  # first node's type tag

    def truncated(rec):
        struct.pack_into("<I", rec, 4, struct.unpack_from("<I", rec, 4)[0] + 1)  # one node too many

    def trailing(rec):
        struct.pack_into("<I", rec, 8, struct.unpack_from("<I", rec, 8)[0] - 1)  # one edge too few

    for case, (fn, want) in {"tag": (bad_tag, "unknown node type tag"), "truncated": (truncated, "binary-format"),
                             "trailing": (trailing, "trailing bytes")}.items():
        arch = _raw_edit(src, str(tmp_path / case), crc, victim, fn)
        assert want in _errors(foundry, load, arch), case

    # a record whose checksum does not match its locator (file digest consistent)
    arch = str(tmp_path / "checksum")
    shutil.copytree(src, arch)
    m = json.load(open(os.path.join(arch, "manifest")))
    raw = bytearray(open(os.path.join(arch, "graphs.bin"), "rb").read())
    i = [l[0] for l in fndg.locators(bytes(raw))].index(victim)
    struct.pack_into("<Q", raw, 10 + 28 * i + 20, struct.unpack_from("<Q", raw, 10 + 28 * i + 20)[0] ^ 1)
    locs = fndg.locators(bytes(raw))
    _commit(arch, m, bytes(raw), locs, crc)
    assert "checksum failure in graph record for label %d" % victim in _errors(foundry, load, arch)


@pytest.mark.parametrize("seed", range(4))
def test_gpu_pack_randomized_members(foundry, archives, oracle, tmp_path, seed):
    """Randomized rewrites of every member of a moe-spmd archive (topology kept):
    kernel names of 5..305 characters (keys longer than the GPU's 92-byte key
    record take the host path; node headers straddle the walk's 8 KiB
    windows), argument blocks of 1 B .. 40 KB (ragged, with u64 lanes inside
    and outside the captured VA range), grids, shared memory, func attrs and
    memcpy / memset records varied per member; patch-entry stubs untouched.
    The GPU-built store equals the offline packer's byte for byte, and the
    fused kernel over it equals the oracle for a random (rank, world, delta)."""
    import random
    src, _ = archives("moe-spmd", b200=False)
    m = manifest(src)
    base, span = m["allocator"]["base"], m["allocator"]["final_offset"]
    stubs = fndg.patch_nodes(open(os.path.join(src, "patch.bin"), "rb").read())
    r = random.Random(seed)
    names = ["k%d_%s" % (i, "n" * r.choice([0, 3, 40, 86, 87, 88, 300])) for i in range(48)]

    def edit(graphs):
        for g in graphs:
            keep = set(stubs.get(g.label, []))
            for n in g.nodes:
                if n.type == 0 and n.id not in keep:
                    if r.random() < 0.5:
                        n.name = r.choice(names)
                    if r.random() < 0.5:
                        size = r.choice([1, 7, 8, 9, 16, 24, 100, 416, 1720, 3001] + [40000] * (r.random() < 0.01))
                        b = bytearray(r.randbytes(size))
                        for off in range(0, size - 7, 8):
                            if r.random() < 0.3:
                                struct.pack_into("<Q", b, off, base + r.randrange(0, span, 8))
                        n.args = bytes(b)
                    if r.random() < 0.3:
                        n.grid = (r.randint(1, 9), r.randint(1, 9), 1)
                    if r.random() < 0.2:
                        n.shmem = r.randint(0, 99999)
                    if r.random() < 0.2:
                        n.fattrs = struct.pack("<6i", *[r.randint(-1, 9) for _ in range(6)])
                elif n.type in (1, 2) and r.random() < 0.3:
                    n.mem = (base + r.randrange(0, span, 16), r.randrange(0, 1 << 64), r.randint(1, 4096))

    arch = _rewrite(src, str(tmp_path / "random"), oracle.crc64, edit)
    _same_store(foundry, arch)
    # and the fused kernel over that store (random rank / world / relocation)
    # equals the oracle's PrepareFn + relocation for every member
    from paper_2604_06664_b200 import capi
    blob, _ = foundry._foundry._pack_store_bytes(arch, True)
    open(os.path.join(arch, "templates.fdt"), "wb").write(blob)  # read by the decoder only
    api = capi.CApi()
    dev = api.device_open(0)
    store = api.store_upload(dev, blob)
    try:
        world = r.choice([1, 2, 4, 8])
        rank = r.randrange(world)
        delta = r.choice([0, 0x10000, 0x10000000000, 0x10000 * r.randrange(1, 1 << 20)])
        members, _ = api.materialize(dev, store, rank, world, base + delta if delta else 0)
        try:
            got = foundry._foundry._decode_member_images(arch, api.members_download(members))
        finally:
            api.lib.fdy_members_free(members)
        want, _ = oracle.materialize_archive(arch, rank, world, delta)
        assert got == want, (rank, world, hex(delta))
    finally:
        api.lib.fdy_store_free(store)
        api.lib.fdy_device_close(dev)


@pytest.mark.parametrize("name,seed", [("micro", 0), ("micro", 1), ("moe-spmd", 2), ("moe-spmd", 3)])
def test_gpu_pack_byte_flip_fuzz(foundry, archives, oracle, tmp_path, name, seed):
    """Random byte flips inside member records (record checksums, locators and
    the file digest kept consistent, so only the decoder / packer can object):
    the GPU packer either builds the offline packer's exact store or raises its
    exact error, for every mutation."""
    import random
    src, _ = archives(name, b200=False)
    raw = open(os.path.join(src, "graphs.bin"), "rb").read()
    locs = fndg.locators(raw)
    r = random.Random(1000 + seed + 7919 * int(os.environ.get("FOUNDRY_FUZZ_ROUND", "0")))
    outcomes = {"store": 0, "error": 0}
    for i in range(int(os.environ.get("FOUNDRY_FUZZ_N", "24"))):
        label, _, length, _ = r.choice(locs)
        flips = [(r.randrange(length), r.randrange(1, 256)) for _ in range(r.choice([1, 1, 2, 4]))]

        def fn(rec, flips=flips):
            for at, x in flips:
                rec[at] ^= x

        arch = _raw_edit(src, str(tmp_path / ("m%d" % i)), oracle.crc64, label, fn)
        try:
            cpu, _ = foundry._foundry._pack_store_bytes(arch, False)
        except foundry.FoundryError as e:
            with pytest.raises(foundry.FoundryError) as gpu:
                foundry._foundry._pack_store_bytes(arch, True)
            assert str(gpu.value) == str(e), (i, label, flips)
            outcomes["error"] += 1
        else:
            gpu, _ = foundry._foundry._pack_store_bytes(arch, True)
            assert gpu == cpu, (i, label, flips, _first_difference(gpu, cpu))
            outcomes["store"] += 1
        shutil.rmtree(arch)
    assert outcomes["error"] > 0


@pytest.mark.parametrize("seed", range(2))
def test_gpu_pack_patch_table_fuzz(foundry, archives, oracle, tmp_path, seed):
    """Random byte flips in patch.bin (manifest digest kept consistent): the GPU
    packer (patch-table view, entries on the GPU) builds the offline packer's
    exact store or raises its exact error."""
    import random
    src, _ = archives("moe-spmd", b200=False)
    patch = open(os.path.join(src, "patch.bin"), "rb").read()
    r = random.Random(2000 + seed + 7919 * int(os.environ.get("FOUNDRY_FUZZ_ROUND", "0")))
    errors = 0
    for i in range(int(os.environ.get("FOUNDRY_FUZZ_N", "24"))):
        arch = str(tmp_path / ("p%d" % i))
        shutil.copytree(src, arch)
        mutated = bytearray(patch)
        for _ in range(r.choice([1, 1, 2, 3])):
            mutated[r.randrange(len(mutated))] ^= r.randrange(1, 256)
        open(os.path.join(arch, "patch.bin"), "wb").write(bytes(mutated))
        m = json.load(open(os.path.join(arch, "manifest")))
        m["files"]["patch.bin"] = oracle.crc64(bytes(mutated))
        json.dump(m, open(os.path.join(arch, "manifest"), "w"))
        try:
            cpu, _ = foundry._foundry._pack_store_bytes(arch, False)
        except foundry.FoundryError as e:
            with pytest.raises(foundry.FoundryError) as gpu:
                foundry._foundry._pack_store_bytes(arch, True)
            assert str(gpu.value) == str(e), i
            errors += 1
        else:
            gpu, _ = foundry._foundry._pack_store_bytes(arch, True)
            assert gpu == cpu, (i, _first_difference(gpu, cpu))
        shutil.rmtree(arch)
    assert errors > 0
