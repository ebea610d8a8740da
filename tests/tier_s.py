"""Tier-S fixtures: model-shaped graphs beyond what the tier-R
workload generator expresses — kernel argument blocks up to 1720 bytes (the
Appendix-B GEMM node, support.hpp:255-305) with embedded device pointers at
8-byte-aligned and unaligned offsets, ragged sizes, and grid dims that vary
between members of a template. Built by rewriting a tier-R archive's graphs
(topology unchanged), with function-level parity only (TEST INFRASTRUCTURE).
"""
from __future__ import annotations

import json
import os
import random
import shutil
import struct

import fndg


def make_tier_s(src: str, dst: str, crc64, seed: int = 7) -> str:
    shutil.copytree(src, dst)
    m = json.load(open(os.path.join(dst, "manifest")))
    base, span = m["allocator"]["base"], m["allocator"]["final_offset"]
    raw = open(os.path.join(dst, "graphs.bin"), "rb").read()
    (version,) = struct.unpack_from("<H", raw, 4)
    graphs = fndg.graphs(raw)
    ext_of = {}  # node id -> its GEMM-block extension (identical across members)
    tail_of = {}
    for g in graphs:
        for n in g.nodes:
            if n.type != 0 or n.name.startswith("stub_"):
                continue
            if n.id % 3 == 0:
                key = (n.id, len(n.args))
                if key not in ext_of:
                    r = random.Random(seed * 1_000_003 + n.id)
                    # GEMM-like block: 1720 bytes (ragged: not a multiple of 16)
                    ext = bytearray(r.randbytes(1720 - len(n.args)))
                    for off in range(0, len(ext) - 8, 24):  # device pointers, some unaligned
                        o = off + (off // 24) % 3  # 8-aligned in the block when (len+o) % 8 == 0
                        struct.pack_into("<Q", ext, o, base + r.randrange(0, span, 16))
                    ext_of[key] = ext
                ext = bytearray(ext_of[key])
                # member-dependent bytes: batch label, a per-batch scratch pointer
                struct.pack_into("<Q", ext, 40, g.label)
                struct.pack_into("<Q", ext, 48, base + 0x10000 * (g.label % 7))
                n.args = n.args + bytes(ext)
            elif n.id % 5 == 0:
                if n.id not in tail_of:
                    tail_of[n.id] = random.Random(seed * 1_000_003 + n.id).randbytes(13)
                n.args = n.args + tail_of[n.id]  # ragged tail
            if n.id % 7 == 0:
                n.grid = (n.grid[0], n.grid[1], 1 + g.label % 3)  # dims differ between members
    data, locs = fndg.write_container(graphs, version, crc64)
    open(os.path.join(dst, "graphs.bin"), "wb").write(data)
    by_label = {l[0]: l for l in locs}
    for grp in m["grouping"]["groups"]:
        grp["locators"] = [list(by_label[l[0]]) for l in grp["locators"]]
    m["files"]["graphs.bin"] = crc64(data)
    m["files"].pop("templates.fdt", None)
    if os.path.exists(os.path.join(dst, "templates.fdt")):
        os.remove(os.path.join(dst, "templates.fdt"))
    json.dump(m, open(os.path.join(dst, "manifest"), "w"))
    return dst


def make_big_smem(src: str, dst: str, crc64) -> str:
    """Every kernel node whose recorded function attribute allows more than
    48 KiB of dynamic shared memory launches with exactly that much (the
    attribute's value). Such a launch is only valid if LOAD restored the
    function's MAX_DYNAMIC_SHARED_SIZE_BYTES on this device."""
    shutil.copytree(src, dst)
    m = json.load(open(os.path.join(dst, "manifest")))
    raw = open(os.path.join(dst, "graphs.bin"), "rb").read()
    (version,) = struct.unpack_from("<H", raw, 4)
    graphs = fndg.graphs(raw)
    big = 0
    for g in graphs:
        for n in g.nodes:
            if n.type == 0:
                (limit,) = struct.unpack_from("<i", n.fattrs, 0)
                if limit > 48 * 1024:
                    n.shmem = limit
                    big += 1
    assert big > 0
    data, locs = fndg.write_container(graphs, version, crc64)
    open(os.path.join(dst, "graphs.bin"), "wb").write(data)
    by_label = {l[0]: l for l in locs}
    for grp in m["grouping"]["groups"]:
        grp["locators"] = [list(by_label[l[0]]) for l in grp["locators"]]
    m["files"]["graphs.bin"] = crc64(data)
    m["files"].pop("templates.fdt", None)
    if os.path.exists(os.path.join(dst, "templates.fdt")):
        os.remove(os.path.join(dst, "templates.fdt"))
    json.dump(m, open(os.path.join(dst, "manifest"), "w"))
    return dst
