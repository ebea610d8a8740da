"""NumPy emulation of the fused materialize kernel over a packed FNDT store.

TEST INFRASTRUCTURE: lets the CPU-only suite check the packer's diff/rank-op
streams end to end (store -> member images -> FNDG records == oracle) without
a GPU. It restates csrc/kernels/materialize.cu, not the reference; the GPU
suite checks the kernel itself against the oracle.
"""
from __future__ import annotations

import struct

import numpy as np

HEADER = struct.Struct("<4sHHIIIIIIII")  # up to n_rank_ops
SEC_NAMES = ["groups", "timages", "cmeta", "members", "tiles", "didx", "ddata",
             "rops", "kernels", "nodeattrs", "edges", "strings"]

TILE_DT = np.dtype([("src_off", "<u8"), ("dst_off", "<u8"), ("nchunks", "<u4"), ("member", "<u4"),
                    ("diff_lo", "<u4"), ("diff_hi", "<u4"), ("rop_lo", "<u4"), ("rop_hi", "<u4"),
                    ("chunk_base", "<u4"), ("pad", "<u4")])
ROP_DT = np.dtype([("chunk", "<u4"), ("kind", "u1"), ("shift", "i1"), ("mask", "<u2"),
                   ("aux", "<u4"), ("pad", "<u4")])


def parse_header(blob: bytes) -> dict:
    f = HEADER.unpack_from(blob, 0)
    h = dict(zip(["magic", "version", "flags", "header_bytes", "n_groups", "n_members",
                  "n_kernels", "n_tiles", "tile_chunks", "n_diffs", "n_rank_ops"], f))
    (h["source_graphs_crc"], h["source_patch_crc"], h["old_base"], h["final_offset"],
     h["real_comm_hash"], h["members_image_bytes"], h["total_nodes"]) = struct.unpack_from("<7Q", blob, 40)
    h["n_plain_tiles"], h["n_values"], h["source_slots_crc"] = struct.unpack_from("<IIQ", blob, 96)
    secs = struct.unpack_from("<%dQ" % (2 * len(SEC_NAMES)), blob, 112)
    h["sec"] = {n: (secs[2 * i], secs[2 * i + 1]) for i, n in enumerate(SEC_NAMES)}
    return h


def expand(blob: bytes, rank: int, world: int, new_base: int = 0, values=()) -> bytes:
    h = parse_header(blob)
    assert h["magic"] == b"FNDT"
    b = np.frombuffer(blob, dtype=np.uint8)

    def sec(name, dtype):
        off, n = h["sec"][name]
        return b[off:off + n].view(dtype)

    tiles = sec("tiles", TILE_DT)
    cmeta = sec("cmeta", np.uint8)
    didx = sec("didx", np.uint16)
    ddata = sec("ddata", np.uint64)
    rops = sec("rops", ROP_DT)
    timg_base = h["sec"]["timages"][0]
    old, span = h["old_base"], h["final_offset"]
    delta = (new_base - old) % (1 << 64) if new_base else 0

    def relocate(chunks, lanes_of):
        lanes = chunks.view("<u8").reshape(-1, 2)
        for lane, bit in ((0, 1), (1, 2)):
            v = lanes[:, lane]
            sel = ((lanes_of & bit) != 0) & ((v - np.uint64(old)) < np.uint64(span))
            v[sel] = v[sel] + np.uint64(delta)

    # K1 once over the template images (the kernel's first grid)
    toff, tn = h["sec"]["timages"]
    timg = b[toff:toff + tn].copy().reshape(-1, 16)
    if delta:
        relocate(timg, cmeta.astype(np.uint32))
    out = np.zeros(h["members_image_bytes"], dtype=np.uint8)
    for t in tiles:
        n = int(t["nchunks"])
        first = (int(t["src_off"]) - timg_base) // 16
        chunks = timg[first:first + n].copy()
        lo, hi = int(t["diff_lo"]), int(t["diff_hi"])
        if hi > lo:  # K2 + K1 on the member's own lanes
            words = didx[lo:hi].astype(np.uint32)
            vals = ddata[lo:hi].copy()
            if delta:
                sel = ((words & 0x8000) != 0) & ((vals - np.uint64(old)) < np.uint64(span))
                vals[sel] = vals[sel] + np.uint64(delta)
            chunks.view("<u8").reshape(-1)[(words & 0x7FFF).astype(np.int64)] = vals
        flat = chunks.reshape(-1)
        for op in rops[int(t["rop_lo"]):int(t["rop_hi"])]:
            kind = int(op["kind"])
            val = {0: rank, 1: world, 2: int(op["aux"])}.get(kind)
            if val is None:
                val = values[int(op["aux"])] if int(op["aux"]) < len(values) else 0
            base = 16 * (int(op["chunk"]) - int(t["chunk_base"]))
            for j in range(16):
                if int(op["mask"]) >> j & 1:
                    flat[base + j] = (val >> (8 * (j - int(op["shift"])))) & 0xFF
        dst = int(t["dst_off"])
        out[dst:dst + 16 * n] = flat
    return out.tobytes()
