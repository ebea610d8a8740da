"""SAVE-side writer parity: archives from this build are byte-identical to the
reference's (golden digests from the reference; live `diff` when oracle/_ref
exists), deterministic, and the spec / tooling surface behaves like the
reference (test_smoke.py, test_workload_gen.cpp, test_pipeline.cpp)."""
from __future__ import annotations

import filecmp
import json
import os
import subprocess

import pytest

from conftest import ROOT, manifest

GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def spec_of(foundry, text):
    return foundry.preset(text) if text in foundry.preset_names() else foundry.workload_from_text(text)


@pytest.mark.parametrize("name", sorted(GOLDEN["archives"]))
def test_save_matches_reference_digests(foundry, oracle, tmp_path, name):
    g = GOLDEN["archives"][name]
    out = str(tmp_path / name)
    outcome = foundry.save(spec_of(foundry, g["spec"]), out, b200_artifacts=False)
    m = manifest(out)
    assert {k: "%016x" % v for k, v in m["files"].items()} == g["files"]
    assert "%016x" % oracle.crc64(open(os.path.join(out, "manifest"), "rb").read()) == g["manifest_crc"]
    traces = "".join("# batch %d\n%s" % (b, t) for b, t in sorted(outcome.traces.items()))
    assert "%016x" % oracle.crc64(traces.encode()) == g["save_traces_crc"]


@pytest.mark.parametrize("preset", ["dense-small", "moe-spmd"])
def test_save_live_byte_identical_to_reference(foundry, ref_tool, tmp_path, preset):
    ours, ref = tmp_path / "ours", tmp_path / "ref"
    outcome = foundry.save(foundry.preset(preset), str(ours), b200_artifacts=False)
    subprocess.run([ref_tool, "save", preset, str(ref), str(tmp_path / "ref.traces")], check=True,
                   capture_output=True)
    cmp = filecmp.dircmp(ours, ref)
    assert not cmp.diff_files and not cmp.left_only and not cmp.right_only
    for rel in ["graphs.bin", "catalog.bin", "patch.bin", "memlayout.bin", "manifest"]:
        assert (ours / rel).read_bytes() == (ref / rel).read_bytes()
    traces = "".join("# batch %d\n%s" % (b, t) for b, t in sorted(outcome.traces.items()))
    assert traces == (tmp_path / "ref.traces").read_text()


def test_two_saves_are_byte_identical_including_b200_artifacts(foundry, tmp_path):
    spec = foundry.preset("micro")
    foundry.save(spec, str(tmp_path / "a"))
    foundry.save(spec, str(tmp_path / "b"))
    files_a = sorted(p.relative_to(tmp_path / "a") for p in (tmp_path / "a").rglob("*") if p.is_file())
    files_b = sorted(p.relative_to(tmp_path / "b") for p in (tmp_path / "b").rglob("*") if p.is_file())
    assert files_a == files_b
    assert any(str(p).endswith(".sm_100a.cubin") for p in files_a)
    assert any(str(p) == "templates.fdt" for p in files_a)
    for rel in files_a:
        assert (tmp_path / "a" / rel).read_bytes() == (tmp_path / "b" / rel).read_bytes()


def test_b200_artifacts_are_recorded_in_the_manifest(foundry, oracle, tmp_path):
    out = str(tmp_path / "m")
    foundry.save(foundry.preset("moe-spmd"), out)
    m = manifest(out)
    assert "templates.fdt" in m["files"]
    cubins = [k for k in m["files"] if k.endswith(".sm_100a.cubin")]
    assert len(cubins) == len([k for k in m["files"] if k.endswith(".bin") and k.startswith("binaries/")])
    for rel, digest in m["files"].items():
        assert oracle.crc64(open(os.path.join(out, rel), "rb").read()) == digest


def test_preset_names_and_spec_round_trip(foundry):
    assert foundry.preset_names() == ["micro", "dense-small", "moe-spmd"]
    assert foundry.preset("micro").batch_max == 8
    with pytest.raises(foundry.FoundryError, match="unknown preset"):
        foundry.preset("nope")
    spec = foundry.preset("moe-spmd")
    text = foundry.spec_text(spec)
    assert foundry.spec_text(foundry.workload_from_text(text)) == text


@pytest.mark.parametrize("text,msg", [
    ("batch_max = 0\n", "batch_max must be >= 1"),
    ("kernels_per_layer = 9\n", "kernels_per_layer must be in"),
    ("thresholds = 5,3\nbatch_max=8\n", "strictly increasing"),
    ("comm = spmd\ncollectives_per_layer = 0\n", "collectives_per_layer >= 1"),
    ("bogus = 1\n", "unknown spec key"),
    ("seed = x\n", "bad value for 'seed'"),
])
def test_spec_violations(foundry, text, msg):
    with pytest.raises(foundry.FoundryError, match="spec-violation: .*" + msg):
        foundry.workload_from_text(text)


def test_save_refuses_non_empty_dirs_and_cleans_up(foundry, tmp_path):
    (tmp_path / "full").mkdir()
    (tmp_path / "full" / "x").write_text("x")
    with pytest.raises(foundry.FoundryError, match="exists and is not empty"):
        foundry.save(foundry.preset("micro"), str(tmp_path / "full"))
    spec = foundry.workload_from_text(foundry.spec_text(foundry.preset("moe-spmd")).replace(
        "emit_raw_collective = 0", "emit_raw_collective = 1"))
    with pytest.raises(foundry.FoundryError, match="unpatchable-comm"):
        foundry.save(spec, str(tmp_path / "raw"))
    assert not (tmp_path / "raw").exists()


def test_inspect_and_diff(foundry, tmp_path):
    out = str(tmp_path / "arch")
    foundry.save(foundry.preset("micro"), out)
    text = foundry.inspect_text(out)
    assert "8 captured, 3 templates" in text
    identical, report = foundry.diff_archives(out, out)
    assert identical and "identical" in report
    doc = foundry.inspect_graph_json(out, 4)
    assert '"function_name"' in doc and '"extra_argBuffer_hex"' in doc
    other = str(tmp_path / "other")
    foundry.save(foundry.preset("dense-small"), other, b200_artifacts=False)
    identical, report = foundry.diff_archives(out, other)
    assert not identical and "workload specs differ" in report


def test_inspect_matches_reference_text(foundry, ref_tool, tmp_path):
    """Tooling output equals the reference module's. The reference pybind module
    runs in a subprocess: both builds bind a C++ `foundry::Error`, and pybind11
    would otherwise share one exception translator between the two modules."""
    import sys
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "foundry_ref")):
        pytest.skip("reference python module not built")
    ours = str(tmp_path / "ours")
    foundry.save(foundry.preset("moe-spmd"), ours, b200_artifacts=False)
    code = ("import sys, json; sys.path.insert(0, %r); import foundry_ref as f; "
            "print(json.dumps([f.inspect_text(%r), f.inspect_graph_json(%r, 37)]))" % (ref_dir, ours, ours))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True).stdout
    ref_inspect, ref_json = json.loads(out)
    assert foundry.inspect_text(ours) == ref_inspect
    assert foundry.inspect_graph_json(ours, 37) == ref_json


def test_pack_archive_matches_the_reference_and_round_trips(foundry, ref_tool, tmp_path):
    """Single-file FNDA archive (reference pack_archive / unpack_archive,
    pipeline.cpp:740-817): byte-identical to the reference's, and unpacking
    restores the directory; corruption and path escapes are archive errors
    (test_pipeline.cpp:360-385)."""
    import filecmp
    import subprocess

    arch = tmp_path / "arch"
    foundry.save(foundry.preset("micro"), str(arch))
    foundry.pack_archive(str(arch), str(tmp_path / "ours.fnda"))
    subprocess.run([ref_tool, "pack", str(arch), str(tmp_path / "ref.fnda")], check=True)
    assert (tmp_path / "ours.fnda").read_bytes() == (tmp_path / "ref.fnda").read_bytes()
    foundry.unpack_archive(str(tmp_path / "ours.fnda"), str(tmp_path / "back"))
    cmp = filecmp.dircmp(arch, tmp_path / "back")
    assert not cmp.left_only and not cmp.right_only and not cmp.diff_files
    assert foundry.diff_archives(str(arch), str(tmp_path / "back"))[0]
    data = bytearray((tmp_path / "ours.fnda").read_bytes())
    data[-5] ^= 1
    (tmp_path / "bad.fnda").write_bytes(bytes(data))
    with pytest.raises(foundry.FoundryError, match="integrity check failed"):
        foundry.unpack_archive(str(tmp_path / "bad.fnda"), str(tmp_path / "bad"))
    with pytest.raises(foundry.FoundryError, match="bad magic"):
        foundry.unpack_archive(str(arch / "graphs.bin"), str(tmp_path / "bad2"))
