"""Pins the C oracle (oracle/foundry_oracle.c) before anything trusts it.

* CRC-64/XZ known answer and bitwise cross-check (reference test_hash.cpp:13-27,
  support.hpp:45-55).
* Golden vectors generated from the compiled reference (tests/golden/golden.json,
  tests/golden/make_golden.py): per-member CRCs of the reference PrepareFn for
  several (rank, world), and the reference replay's verdict on relocated members.
* Live comparison with the reference itself when oracle/_ref is built.
"""
from __future__ import annotations

import json
import os
import random
import subprocess

import pytest

import fndg
from conftest import ROOT, manifest

GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def test_crc64_check_value(oracle):
    assert oracle.crc64(b"123456789") == 0x995DC9BBDF1939FA
    assert "%016x" % oracle.crc64(b"123456789") == GOLDEN["crc64_check"]["123456789"]
    assert oracle.crc64(b"") == 0


def test_crc64_table_matches_bitwise(oracle):
    rng = random.Random(5)
    for n in (1, 7, 8, 9, 63, 64, 65, 1000, 4097):
        data = bytes(rng.randrange(256) for _ in range(n))
        assert oracle.crc64(data) == oracle.crc64_bitwise(data)


def golden_archive(foundry, tmp_path, name):
    spec_text = GOLDEN["archives"][name]["spec"]
    spec = foundry.preset(spec_text) if spec_text in foundry.preset_names() else foundry.workload_from_text(spec_text)
    out = str(tmp_path / name)
    foundry.save(spec, out, b200_artifacts=False)
    return out


@pytest.mark.parametrize("name", sorted(GOLDEN["archives"]))
def test_oracle_matches_reference_golden_members(foundry, oracle, tmp_path, name):
    arch = golden_archive(foundry, tmp_path, name)
    g = GOLDEN["archives"][name]
    for case in g["cases"]:
        data, nreloc = oracle.materialize_archive(arch, case["rank"], case["world"], case["delta"])
        assert "%016x" % oracle.crc64(data) == case["container_crc"], case
        recs = {str(k): "%016x" % oracle.crc64(v) for k, v in fndg.records(data).items()}
        assert recs == case["records"]
        if case["delta"]:
            assert nreloc == case["relocated_slots"]


def test_oracle_live_against_reference_prepare(oracle, ref_tool, tmp_path):
    arch = str(tmp_path / "moe")
    subprocess.run([ref_tool, "save", "moe-spmd", arch], check=True, capture_output=True)
    for rank, world in [(0, 1), (5, 8)]:
        prep = str(tmp_path / "prep.fndg")
        subprocess.run([ref_tool, "prepare", arch, str(rank), str(world), prep], check=True)
        ours, _ = oracle.materialize_archive(arch, rank, world)
        assert ours == open(prep, "rb").read()


def test_oracle_relocation_accepted_by_reference_replay(oracle, ref_tool, tmp_path):
    """No reference function relocates; the reference's simulated replay (which
    knows the true hidden pointer offsets) must accept the relocated members at
    the shifted base and report every address moved by exactly delta."""
    arch = str(tmp_path / "moe")
    subprocess.run([ref_tool, "save", "moe-spmd", arch], check=True, capture_output=True)
    # one granule, the 0x7000.. -> 0x7100.. pair of test_smoke.py, and a
    # SplitMix64(0xF00D)-drawn granule-aligned delta < 2^40
    z = (0xF00D + 0x9E3779B97F4A7C15) & (2**64 - 1)
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    z ^= z >> 31
    drawn = (z % (1 << 40)) & ~0xFFFF
    base_traces = str(tmp_path / "t0")
    prep = str(tmp_path / "p0.fndg")
    subprocess.run([ref_tool, "prepare", arch, "1", "4", prep], check=True)
    subprocess.run([ref_tool, "replay", arch, prep, "0", base_traces], check=True)
    t0 = open(base_traces).read().splitlines()
    for delta in (0x10000, 0x10000000000, drawn):
        data, nreloc = oracle.materialize_archive(arch, 1, 4, delta)
        moved = str(tmp_path / "reloc.fndg")
        open(moved, "wb").write(data)
        out = str(tmp_path / "t1")
        r = subprocess.run([ref_tool, "replay", arch, moved, "%x" % delta, out], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        t1 = open(out).read().splitlines()
        assert len(t0) == len(t1)
        for a, b in zip(t0, t1):
            if a.startswith("#"):
                assert a == b
                continue
            aa, ab = a.split(" addrs=")[1], b.split(" addrs=")[1]
            xs = [int(x, 16) for x in aa.split(",") if x]
            ys = [int(x, 16) for x in ab.split(",") if x]
            assert [x + delta for x in xs] == ys
        # zero false positives on tier-R data: exactly the true address fields move
        m = manifest(arch)
        per_graph = 12 * 8 * 5 + 24 + 3  # kernel address fields + stub buffers + memops
        assert nreloc == per_graph * m["grouping"]["total"]
    # unrelocated members at a shifted base are rejected by the reference
    r = subprocess.run([ref_tool, "replay", arch, prep, "10000", str(tmp_path / "bad")],
                       capture_output=True, text=True)
    assert r.returncode == 3 and "unmapped-address" in r.stderr


def test_oracle_error_behaviour(oracle, foundry, tmp_path):
    from oracle_lib import OracleError

    arch = golden_archive(foundry, tmp_path, "moe-small")
    with pytest.raises(OracleError, match="rank 4 is outside world size 4"):
        oracle.materialize_archive(arch, 4, 4)
    graphs = bytearray(open(os.path.join(arch, "graphs.bin"), "rb").read())
    lab, off, ln, _ = fndg.locators(bytes(graphs))[3]
    graphs[off + ln // 2] ^= 0x40
    m = manifest(arch)
    patch = open(os.path.join(arch, "patch.bin"), "rb").read()
    with pytest.raises(OracleError, match="checksum failure in graph record for label %d" % lab):
        oracle.materialize(bytes(graphs), patch, m["comm"]["real_binary_hash"], 0, 1,
                           m["allocator"]["base"], m["allocator"]["final_offset"])
    with pytest.raises(OracleError, match="no real comm binary"):
        oracle.materialize(open(os.path.join(arch, "graphs.bin"), "rb").read(), patch, 0, 0, 1,
                           m["allocator"]["base"], m["allocator"]["final_offset"])
