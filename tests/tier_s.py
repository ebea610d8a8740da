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
    for g in graphs:
        for n in g.nodes:
            if n.type != 0 or n.name.startswith("stub_"):
                continue
            r = random.Random(seed * 1_000_003 + n.id)  # same per node across members
            if n.id % 3 == 0:
                # GEMM-like block: 1720 bytes (ragged: not a multiple of 16)
                ext = bytearray(r.getrandbits(8) for _ in range(1720 - len(n.args)))
                for off in range(0, len(ext) - 8, 24):  # device pointers, some unaligned
                    p = base + r.randrange(0, span, 16)
                    o = off + (off // 24) % 3  # 8-aligned in the block when (len+o) % 8 == 0
                    struct.pack_into("<Q", ext, o, p)
                # member-dependent bytes: batch label, a per-batch scratch pointer
                struct.pack_into("<Q", ext, 40, g.label)
                struct.pack_into("<Q", ext, 48, base + 0x10000 * (g.label % 7))
                n.args = n.args + bytes(ext)
            elif n.id % 5 == 0:
                n.args = n.args + bytes(r.getrandbits(8) for _ in range(13))  # ragged tail
            if n.id % 7 == 0:
                n.grid = (n.grid[0], n.grid[1], 1 + g.label % 3)  # dims differ between members
    data, locs = fndg.write_container(graphs, version, crc64)
    open(os.path.join(dst, "graphs.bin"), "wb").write(data)
    by_label = {l[0]: l for l in locs}
    for grp in m["grouping"]["groups"]:
        grp["locators"] = [list(by_label[l[0]]) for l in grp["locators"]]
    m["files"]["graphs.bin"] = crc64(data)
    m["files"].pop("templates.fdt", None)
    os.remove(os.path.join(dst, "templates.fdt"))
    json.dump(m, open(os.path.join(dst, "manifest"), "w"))
    return dst
