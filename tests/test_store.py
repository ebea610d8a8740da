"""Template-store packer (FNDT) checked end to end on CPU: pack -> NumPy
emulation of the fused kernel -> decode -> byte-identical to the oracle."""
from __future__ import annotations

import os
import struct

import numpy as np
import pytest

import store_emulator as emu
from conftest import manifest


def emulate(foundry, arch, rank, world, delta=0, values=()):
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    m = manifest(arch)
    nb = m["allocator"]["base"] + delta if delta else 0
    arena = emu.expand(blob, rank, world, nb, values)
    return foundry._foundry._decode_member_images(arch, arena)


@pytest.mark.parametrize("name,cases", [
    ("micro", [(0, 1, 0), (0, 1, 0x10000)]),
    ("llama3-8b", [(0, 1, 0), (0, 1, 0x123450000)]),
    ("moe-spmd", [(0, 1, 0), (1, 4, 0), (7, 8, 0x10000000000), (2, 3, 0x10000)]),
])
def test_store_expansion_equals_oracle(foundry, oracle, archives, name, cases):
    arch, _ = archives(name)
    for rank, world, delta in cases:
        want, _ = oracle.materialize_archive(arch, rank, world, delta)
        assert emulate(foundry, arch, rank, world, delta) == want, (rank, world, hex(delta))


def test_store_header_describes_the_archive(foundry, archives):
    from paper_2604_06664_b200 import capi
    arch, outcome = archives("moe-spmd")
    m = manifest(arch)
    h = capi.store_header(open(os.path.join(arch, "templates.fdt"), "rb").read())
    assert h["n_members"] == outcome.total_graphs == 512
    assert h["n_groups"] == outcome.template_count
    assert h["old_base"] == m["allocator"]["base"]
    assert h["final_offset"] == m["allocator"]["final_offset"]
    assert h["real_comm_hash"] == m["comm"]["real_binary_hash"]
    assert h["source_graphs_crc"] == m["files"]["graphs.bin"]
    assert h["source_patch_crc"] == m["files"]["patch.bin"]
    assert h["tile_chunks"] == 1024
    # 12 layers x 2 collectives -> 24 patch entries per graph, each: rank + world
    # (one op each, 8-byte aligned inside a chunk); the kernel swap is folded
    # into the images. Every member of a group patches the same offsets, so a
    # group's op ranges are stored once and shared by its members' tiles.
    assert h["n_rank_ops"] == h["n_groups"] * 24 * 2
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    off, n = h["sec"]["tiles"]
    tiles = np.frombuffer(blob, emu.TILE_DT, n // emu.TILE_DT.itemsize, off)
    assert int((tiles["rop_hi"] - tiles["rop_lo"]).sum()) == 512 * 24 * 2
    alg = capi.algorithmic_bytes(h)
    assert alg["write"] == h["members_image_bytes"] and alg["read"] > 0


def test_store_is_smaller_than_graphs_bin(archives):
    arch, _ = archives("moe-spmd")
    store = os.path.getsize(os.path.join(arch, "templates.fdt"))
    graphs = os.path.getsize(os.path.join(arch, "graphs.bin"))
    assert store < graphs / 3


def test_repacking_is_deterministic(foundry, archives, tmp_path):
    import shutil
    arch, _ = archives("micro")
    copy = tmp_path / "copy"
    shutil.copytree(arch, copy)
    foundry._foundry._pack_store(str(copy))
    assert (copy / "templates.fdt").read_bytes() == open(os.path.join(arch, "templates.fdt"), "rb").read()


def test_pack_rejects_a_patch_on_a_non_stub(foundry, archives, tmp_path):
    """apply_rank_patches raises archive-corruption for a patch entry whose node
    is not the recorded stub (rank_forge.cpp:141-143); the packer does too."""
    import shutil
    arch, _ = archives("moe-spmd", b200=False)
    bad = tmp_path / "bad"
    shutil.copytree(arch, bad)
    patch = bytearray((bad / "patch.bin").read_bytes())
    # first entry: magic(4) ver(2) placeholder(8) ngraphs(4) label(4) count(4) node_id(4)
    struct.pack_into("<I", patch, 26, 1)  # point it at node 1 (a compute kernel)
    (bad / "patch.bin").write_bytes(bytes(patch))
    with pytest.raises(foundry.FoundryError, match="archive-corruption: node 1 is not the recorded stub"):
        foundry._foundry._pack_store(str(bad))


def test_error_quoting_non_utf8_bytes_is_a_foundry_error(foundry, archives, tmp_path):
    """A corrupt stub name in patch.bin (bytes 0xff) reaches the error message;
    FoundryError still carries it (backslash-escaped) instead of the binding
    failing to decode it (found by tests/test_gpu_pack.py's patch-table fuzz)."""
    import shutil
    arch, _ = archives("moe-spmd", b200=False)
    bad = tmp_path / "bad"
    shutil.copytree(arch, bad)
    patch = bytearray((bad / "patch.bin").read_bytes())
    at = patch.index(b"stub_allreduce")
    patch[at:at + 4] = b"\xff\xfe\xff\xfe"
    (bad / "patch.bin").write_bytes(bytes(patch))
    with pytest.raises(foundry.FoundryError, match=r"\\xff\\xfe"):
        foundry._foundry._pack_store(str(bad))


def test_crc64_host_matches_the_oracle_and_combines(foundry, oracle):
    import random
    rng = random.Random(3)
    for n in (0, 1, 7, 8, 9, 100, 4096, 70001):
        a = bytes(rng.randrange(256) for _ in range(n))
        b = bytes(rng.randrange(256) for _ in range(n // 3 + 1))
        assert foundry._foundry._crc64(a) == oracle.crc64(a)
        combined = foundry._foundry._crc64_combine(oracle.crc64(a), oracle.crc64(b), len(b))
        assert combined == oracle.crc64(a + b)


def test_crc64_folding_paths_match_the_oracle(foundry, oracle):
    # lengths around the 64-byte (PCLMULQDQ) and 256-byte (VPCLMULQDQ, >= 1 KiB)
    # fold boundaries, unaligned starts, and a multi-MiB buffer
    import random
    rng = random.Random(11)
    big = rng.randbytes(3 << 20)
    for n in (255, 256, 257, 1023, 1024, 1025, 1279, 1280, 4095, 65536 + 17, 1 << 20, 3 << 20):
        for off in (0, 1, 13):
            a = big[off:off + n]
            assert foundry._foundry._crc64(a) == oracle.crc64(a), (n, off)


@pytest.fixture(scope="module")
def tier_s_archive(foundry, oracle, archives, tmp_path_factory):
    import tier_s
    src, _ = archives("moe-spmd")
    dst = str(tmp_path_factory.mktemp("tier_s") / "moe-s")
    tier_s.make_tier_s(src, dst, oracle.crc64)
    foundry._foundry._pack_store(dst)
    return dst


@pytest.mark.parametrize("rank,world,delta", [(0, 1, 0), (1, 4, 0x10000), (7, 8, 0x10000000000)])
def test_tier_s_store_expansion_equals_oracle(foundry, oracle, tier_s_archive, rank, world, delta):
    """Model-shaped graphs beyond tier R (1720-byte argument blocks with
    pointers at aligned and unaligned offsets, ragged sizes, grid dims that vary
    inside a template): pack + kernel emulation == oracle."""
    want, _ = oracle.materialize_archive(tier_s_archive, rank, world, delta)
    assert emulate(foundry, tier_s_archive, rank, world, delta) == want


def test_manifest_fast_reader_agrees_or_defers(foundry, archives):
    # parse_manifest reads the manifest with a minimal JSON reader first and hands
    # anything outside its subset to the full JSON parser; it must never disagree
    agrees = foundry._foundry._manifest_fast_path_agrees
    texts = []
    for name, b200 in (("micro", True), ("moe-spmd", True), ("moe-spmd", False)):
        arch, _ = archives(name, b200=b200)
        texts.append(open(os.path.join(arch, "manifest")).read())
    for t in texts:
        assert agrees(t) == 1  # every writer's manifest takes the fast path
    t = texts[0]
    variants = [
        t.replace('"format_version": 1', '"format_version": 1.0', 1),
        t.replace('"kv_cache_bytes": ', '"kv_cache_bytes": -', 1),
        t.replace('{', '{"catalog": "x", ', 1),            # duplicate key
        t.replace('"catalog.bin"', '"catalog\\u002ebin"', 1),  # \u escape
        t.replace('"catalog.bin"', '"catalogé.bin"', 1),  # non-ASCII
        t + " x",                                            # trailing garbage
        t.replace('"patch_table"', '"patch_tablex"', 1),     # missing field
        t.replace('"workload_digest": ', '"workload_digest": 0', 1),  # leading zero
        " \n" + t + "\n ",                                    # whitespace only
    ]
    for v in variants:
        assert agrees(v) in (-1, 1), v[:80]
    assert agrees(variants[-1]) == 1
    for v in variants[:8]:
        assert agrees(v) == -1


# ------------------------------------------------------------------ comm slots

def _with_slots(foundry, archives, tmp_path, table_fn, name="moe-spmd"):
    import shutil

    import comm_slots
    arch, _ = archives(name)
    copy = str(tmp_path / (name + "-slots"))
    shutil.copytree(arch, copy)
    foundry.write_comm_slots(copy, comm_slots.N_VALUES, table_fn(copy))
    return copy


def test_comm_slots_store_expansion_equals_oracle(foundry, oracle, archives, tmp_path):
    """K3 value ops (comm handles, peer buffers): every rank of W=8 gets its own
    value table; writes straddle 16-byte chunks, overlap the rank/world bytes
    (slots apply after them) and use 1/4/8-byte widths."""
    import comm_slots
    from paper_2604_06664_b200 import capi
    arch = _with_slots(foundry, archives, tmp_path, comm_slots.stress_table)
    h = capi.store_header(open(os.path.join(arch, "templates.fdt"), "rb").read())
    m = manifest(arch)
    assert h["n_values"] == comm_slots.N_VALUES
    assert h["source_slots_crc"] == m["files"]["comm_slots.bin"]
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read()
    off, n = h["sec"]["rops"]
    rops = np.frombuffer(blob, emu.ROP_DT, n // emu.ROP_DT.itemsize, off)
    assert (rops["kind"] == 3).any()  # FDT_ROP_VALUE
    outs = set()
    for rank, delta in [(0, 0), (3, 0x10000), (7, 0x10000000000)]:
        vals = comm_slots.rank_values(rank)
        want, _ = oracle.materialize_archive(arch, rank, 8, delta, values=vals)
        assert emulate(foundry, arch, rank, 8, delta, vals) == want, rank
        outs.add(want)
    assert len(outs) == 3


def test_comm_slots_oracle_differs_from_the_reference_only_at_slot_bytes(foundry, oracle, archives, tmp_path,
                                                                       ref_tool):
    """Pin of the slot rule: the oracle with comm slots equals the reference's
    own PrepareFn output (ref_tool prepare) except at exactly the slot bytes,
    which hold the rank's values little-endian."""
    import subprocess

    import comm_slots
    import fndg
    arch = _with_slots(foundry, archives, tmp_path, comm_slots.stress_table)
    rank, vals = 5, comm_slots.rank_values(5)
    got, _ = oracle.materialize_archive(arch, rank, 8, values=vals)
    ref = str(tmp_path / "ref.fndg")
    subprocess.run([ref_tool, "prepare", arch, str(rank), "8", ref], check=True)
    want = {g.label: g for g in fndg.graphs(open(ref, "rb").read())}
    table = comm_slots.stress_table(arch)
    touched = 0
    for g in fndg.graphs(got):
        r = want[g.label]
        expect = {n.id: bytearray(n.args) for n in r.nodes}
        for node, off, idx, width in table.get(g.label, []):
            expect[node][off:off + width] = vals[idx].to_bytes(8, "little")[:width]
            touched += 1
        for a, b in zip(g.nodes, r.nodes):
            assert (a.type, a.grid, a.block, a.hash, a.name) == (b.type, b.grid, b.block, b.hash, b.name)
            assert a.args == bytes(expect[a.id]), (g.label, a.id)
    assert touched > 0


def test_comm_slots_are_validated(foundry, archives, tmp_path):
    """Slots may only name patched comm nodes, must fit the argument buffer,
    and index the value table (archive-corruption / invalid-argument)."""
    import shutil

    import fndg
    arch, _ = archives("moe-spmd")
    copy = str(tmp_path / "bad")
    shutil.copytree(arch, copy)
    nodes = fndg.patch_nodes(open(os.path.join(copy, "patch.bin"), "rb").read())
    label, ids = next(iter(nodes.items()))
    compute = next(i for i in range(1, 50) if i not in ids)
    with pytest.raises(foundry.FoundryError, match="not a patched comm node"):
        foundry.write_comm_slots(copy, 2, {label: [(compute, 0, 0, 8)]})
    with pytest.raises(foundry.FoundryError, match="outside the argument buffer"):
        foundry.write_comm_slots(copy, 2, {label: [(ids[0], 30, 0, 8)]})
    with pytest.raises(foundry.FoundryError, match="value index 2 is outside"):
        foundry.write_comm_slots(copy, 2, {label: [(ids[0], 16, 2, 8)]})
    with pytest.raises(foundry.FoundryError, match="width 9"):
        foundry.write_comm_slots(copy, 2, {label: [(ids[0], 16, 0, 9)]})
    # nothing was written by the failed calls
    assert not os.path.exists(os.path.join(copy, "comm_slots.bin"))
    assert "comm_slots.bin" not in manifest(copy)["files"]


def test_patch_view_equals_the_patch_table(foundry, archives):
    """The zero-copy patch-table view LOAD and the GPU packer read
    (parse_patch_view) yields exactly parse_patch_table's entries, and the same
    error for every truncation of the bytes (reference rank_forge.cpp:43-102)."""
    arch, _ = archives("moe-spmd")
    raw = open(os.path.join(arch, "patch.bin"), "rb").read()
    assert foundry._foundry._patch_view_matches_table(raw)
    for cut in (0, 3, 5, 13, 17, 40, len(raw) // 2, len(raw) - 1):
        with pytest.raises(foundry.FoundryError) as table:
            foundry._foundry._patch_view_matches_table(raw[:cut])
        with pytest.raises(foundry.FoundryError) as view:
            foundry._foundry._parse_patch_view(raw[:cut])
        assert str(table.value) == str(view.value), cut
    with pytest.raises(foundry.FoundryError, match="trailing bytes in patch table"):
        foundry._foundry._parse_patch_view(raw + b"\0")


def test_patch_view_fuzz_matches_the_patch_table(foundry, archives):
    """Random byte flips of a patch table large enough for the two-pass parallel
    view (sizes walked first, graphs decoded on the worker pool): the view
    either equals parse_patch_table's result or raises its exact error."""
    import random
    arch, _ = archives("moe-spmd")
    raw = open(os.path.join(arch, "patch.bin"), "rb").read()
    assert len(raw) >= 256 << 10  # the parallel path
    r = random.Random(7)
    for i in range(200):
        b = bytearray(raw)
        for _ in range(r.choice([1, 2, 3])):
            # length and count fields sit in the first bytes of every entry: aim some flips there
            at = r.randrange(len(b)) if r.random() < 0.5 else r.randrange(min(len(b), 4096))
            b[at] ^= r.randrange(1, 256)
        b = bytes(b)
        try:
            same = foundry._foundry._patch_view_matches_table(b)
        except foundry.FoundryError as e:
            with pytest.raises(foundry.FoundryError) as view:
                foundry._foundry._parse_patch_view(b)
            assert str(view.value) == str(e), i
        else:
            assert same, i


def test_pack_error_is_the_first_failing_member_not_the_first_in_time(foundry, oracle, archives, tmp_path):
    """Two members of a group with different patch errors: the offline packer used to
    report whichever of its threads failed first, so it disagreed with the GPU packer
    (which checks members in order) on some runs; found by the GPU packer's patch-table
    fuzz (tests/test_gpu_pack.py, FOUNDRY_FUZZ_ROUND=5, seed 0, mutation 49). The
    failure is now the lowest failing member's on every run."""
    import json
    import random
    import shutil
    src, _ = archives("moe-spmd", b200=False)
    patch = open(os.path.join(src, "patch.bin"), "rb").read()
    r = random.Random(2000 + 0 + 7919 * 5)  # the fuzz's draw sequence up to mutation 49
    for _ in range(50):
        mutated = bytearray(patch)
        for _ in range(r.choice([1, 1, 2, 3])):
            mutated[r.randrange(len(mutated))] ^= r.randrange(1, 256)
    arch = str(tmp_path / "two-bad-members")
    shutil.copytree(src, arch)
    open(os.path.join(arch, "patch.bin"), "wb").write(bytes(mutated))
    m = json.load(open(os.path.join(arch, "manifest")))
    m["files"]["patch.bin"] = oracle.crc64(bytes(mutated))
    json.dump(m, open(os.path.join(arch, "manifest"), "w"))
    seen = set()
    for _ in range(8):
        with pytest.raises(foundry.FoundryError) as e:
            foundry._foundry._pack_store_bytes(arch, False)
        seen.add(str(e.value))
    assert len(seen) == 1, seen
    assert seen.pop().startswith("archive-corruption: node 29 is not the recorded stub")
