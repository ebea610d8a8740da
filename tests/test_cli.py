"""The `foundry` CLI (paper_2604_06664_b200/foundry) against the reference's
CLI tests (proj/tests/python/test_smoke.py:99-178): same subcommands, output
lines, exit codes and FOUNDRY_BASE_ADDR behaviour."""
from __future__ import annotations

import filecmp
import os
import subprocess

import pytest

from conftest import ROOT

CLI = os.path.join(ROOT, "paper_2604_06664_b200", "foundry")


def run(*args, env=None):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, env=env)


def test_cli_save_inspect_diff(native_build, tmp_path):
    arch = tmp_path / "arch"
    save = run("save", "--workload", "micro", "--out", arch, "--traces", tmp_path / "t.txt")
    assert save.returncode == 0, save.stderr
    assert "3 templates" in save.stdout and (tmp_path / "t.txt").stat().st_size > 0
    inspect = run("inspect", arch)
    assert inspect.returncode == 0 and "templates" in inspect.stdout
    graph = run("inspect", arch, "--graph", 2)
    assert graph.returncode == 0 and graph.stdout.lstrip().startswith("{")
    diff = run("diff", arch, arch)
    assert diff.returncode == 0 and "identical" in diff.stdout
    other = tmp_path / "other"
    assert run("save", "--workload", "dense-small", "--out", other).returncode == 0
    assert run("diff", arch, other).returncode == 1


def test_cli_archives_equal_the_bindings(native_build, foundry, tmp_path):
    """test_cross_process_determinism (test_smoke.py:131-145)."""
    assert run("save", "--workload", "micro", "--out", tmp_path / "cli").returncode == 0
    foundry.save(foundry.preset("micro"), str(tmp_path / "lib"))
    files = sorted(p.relative_to(tmp_path / "cli") for p in (tmp_path / "cli").rglob("*") if p.is_file())
    assert files == sorted(p.relative_to(tmp_path / "lib") for p in (tmp_path / "lib").rglob("*") if p.is_file())
    for rel in files:
        assert (tmp_path / "cli" / rel).read_bytes() == (tmp_path / "lib" / rel).read_bytes()


def test_cli_base_addr_env_and_usage_errors(native_build, tmp_path):
    env = dict(os.environ, FOUNDRY_BASE_ADDR="0x7f0000000000")
    arch = tmp_path / "arch"
    assert run("save", "--workload", "micro", "--out", arch, env=env).returncode == 0
    assert "0x00007f0000000000" in run("inspect", arch).stdout
    assert run("bogus").returncode == 2
    assert run("save", "--workload", "micro").returncode == 2          # --out missing
    bad = run("save", "--workload", "no-such-preset", "--out", tmp_path / "x")
    assert bad.returncode != 0 and "error:" in bad.stderr


@pytest.mark.gpu
def test_cli_round_trip_and_exit_codes(native_build, tmp_path):
    """test_cli_round_trip + test_cli_exit_codes (test_smoke.py:102-162)."""
    arch = tmp_path / "arch"
    assert run("save", "--workload", "micro", "--out", arch, "--traces", tmp_path / "save.txt").returncode == 0
    load = run("load", "--archive", arch, "--replay-all", "--traces", tmp_path / "load.txt")
    assert load.returncode == 0, load.stderr
    assert "8 batch sizes servable" in load.stdout and "replayed 8 graphs" in load.stdout
    assert filecmp.cmp(tmp_path / "save.txt", tmp_path / "load.txt", shallow=False)
    # the B200 modes replay the same traces
    for flag in ("--share-execs", "--device-updates"):
        res = run("load", "--archive", arch, flag, "--replay-all", "--traces", tmp_path / "m.txt")
        assert res.returncode == 0, res.stderr
        assert filecmp.cmp(tmp_path / "save.txt", tmp_path / "m.txt", shallow=False)
    # the manifest wins at LOAD even if the environment disagrees
    env = dict(os.environ, FOUNDRY_BASE_ADDR="0x710000000000")
    assert run("load", "--archive", arch, "--replay-all", env=env).returncode == 0
    # a corrupted payload byte: archive errors exit with 2
    g = arch / "graphs.bin"
    data = bytearray(g.read_bytes())
    data[len(data) // 2] ^= 1
    g.write_bytes(bytes(data))
    broken = run("load", "--archive", arch)
    assert broken.returncode == 2 and "archive" in broken.stderr
