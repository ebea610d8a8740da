"""Pure-Python readers for the archive formats (TEST INFRASTRUCTURE).

Independent of the product's C++ codecs: FNDG graph containers (reference
graph_model.cpp:96-303), FNDB kernel images (kernel_image.cpp:14-90) and the
reference LaunchTrace text (sim_driver.cpp:21-38, replay :402-479), used to
derive expected replay traces from oracle-materialized records.
"""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass, field

TYPES = {0: "KernelNode", 1: "MemcpyNode", 2: "MemsetNode", 3: "EmptyNode"}


@dataclass
class Node:
    id: int
    type: int
    attrs: bytes = b""
    grid: tuple = (1, 1, 1)
    block: tuple = (1, 1, 1)
    shmem: int = 0
    hash: int = 0
    name: str = ""
    fattrs: bytes = b""
    args: bytes = b""
    mem: tuple = (0, 0, 0)


@dataclass
class Graph:
    label: int
    nodes: list = field(default_factory=list)
    edges: list = field(default_factory=list)


def locators(buf: bytes):
    assert buf[:4] == b"FNDG"
    (ver,) = struct.unpack_from("<H", buf, 4)
    (count,) = struct.unpack_from("<I", buf, 6)
    out = []
    for i in range(count):
        out.append(struct.unpack_from("<IQQQ", buf, 10 + 28 * i))
    return out


def decode_record(rec: bytes) -> Graph:
    label, nn, ne = struct.unpack_from("<III", rec, 0)
    at = 12
    g = Graph(label)
    for i in range(nn):
        t = rec[at]
        at += 1
        n = Node(i, t)
        if t == 0:
            n.attrs = rec[at:at + 25]
            at += 25
            dims = struct.unpack_from("<7I", rec, at)
            at += 28
            n.grid, n.block, n.shmem = dims[0:3], dims[3:6], dims[6]
            (n.hash,) = struct.unpack_from("<Q", rec, at)
            at += 8
            (ln,) = struct.unpack_from("<I", rec, at)
            at += 4
            n.name = rec[at:at + ln].decode()
            at += ln
            n.fattrs = rec[at:at + 24]
            at += 24
            (al,) = struct.unpack_from("<I", rec, at)
            at += 4
            n.args = rec[at:at + al]
            at += al
        elif t in (1, 2):
            n.mem = struct.unpack_from("<3Q", rec, at)
            at += 24
        g.nodes.append(n)
    for i in range(ne):
        g.edges.append(struct.unpack_from("<II", rec, at))
        at += 8
    assert at == len(rec)
    return g


def graphs(buf: bytes):
    return [decode_record(buf[off:off + ln]) for (_, off, ln, _) in locators(buf)]


def records(buf: bytes):
    return {lab: buf[off:off + ln] for (lab, off, ln, _) in locators(buf)}


def kernel_image(payload: bytes):
    """FNDB -> {name: (arg_size, hidden_offsets)} (kernel_image.cpp:44-90)."""
    assert payload[:4] == b"FNDB"
    at = 7
    _tag, count = struct.unpack_from("<II", payload, at)
    at += 8
    out = {}
    for _ in range(count):
        (ln,) = struct.unpack_from("<I", payload, at)
        at += 4
        name = payload[at:at + ln].decode()
        at += ln
        size, k = struct.unpack_from("<II", payload, at)
        at += 8
        hidden = list(struct.unpack_from("<%dI" % k, payload, at))
        at += 4 * k + 24
        out[name] = (size, hidden)
    return out


def hidden_map(archive: str):
    """(hash, name) -> hidden offsets, for every binary of an archive."""
    out = {}
    bdir = os.path.join(archive, "binaries")
    for f in os.listdir(bdir):
        if f.endswith(".bin"):
            h = int(f[:16], 16)
            for name, (_, hidden) in kernel_image(open(os.path.join(bdir, f), "rb").read()).items():
                out[(h, name)] = hidden
    return out


def trace_text(g: Graph, hidden, crc64) -> str:
    """Expected replay trace of one prepared graph (sim_driver.cpp:21-38,402-479)."""
    lines = []
    for n in g.nodes:
        s = "node=%d type=%s" % (n.id, TYPES[n.type])
        addrs = []
        if n.type == 0:
            s += " name=%s grid=%d,%d,%d block=%d,%d,%d shmem=%d" % (
                (n.name,) + tuple(n.grid) + tuple(n.block) + (n.shmem,))
            for off in hidden[(n.hash, n.name)]:
                (a,) = struct.unpack_from("<Q", n.args, off)
                addrs.append(a)
            digest = crc64(n.args)
        elif n.type == 1:
            addrs = [n.mem[0], n.mem[1]]
            digest = crc64(struct.pack("<3Q", *n.mem))
        elif n.type == 2:
            addrs = [n.mem[0]]
            digest = crc64(struct.pack("<3Q", *n.mem))
        else:
            digest = 0
        s += " args=%016x addrs=%s" % (digest, ",".join("0x%016x" % a for a in addrs))
        lines.append(s + "\n")
    return "".join(lines)


# ---- writers (tier-S fixtures: model-shaped graphs the tier-R generator cannot express)

def encode_record(g: Graph) -> bytes:
    """Inverse of decode_record (graph_model.cpp:205-218 layout)."""
    out = [struct.pack("<III", g.label, len(g.nodes), len(g.edges))]
    for n in g.nodes:
        out.append(bytes([n.type]))
        if n.type == 0:
            name = n.name.encode()
            out.append(n.attrs)
            out.append(struct.pack("<7I", *n.grid, *n.block, n.shmem))
            out.append(struct.pack("<QI", n.hash, len(name)) + name)
            out.append(n.fattrs)
            out.append(struct.pack("<I", len(n.args)) + n.args)
        elif n.type in (1, 2):
            out.append(struct.pack("<3Q", *n.mem))
    for e in g.edges:
        out.append(struct.pack("<II", *e))
    return b"".join(out)


def write_container(graph_list, version: int, crc64) -> tuple[bytes, list]:
    """FNDG container (graph_model.cpp:244-269): header, 28-byte locators
    {u32 label, u64 offset, u64 length, u64 crc64(record)}, records.
    Returns (bytes, locators)."""
    recs = [encode_record(g) for g in graph_list]
    at = 10 + 28 * len(recs)
    locs = []
    for g, r in zip(graph_list, recs):
        locs.append((g.label, at, len(r), crc64(r)))
        at += len(r)
    head = b"FNDG" + struct.pack("<HI", version, len(recs))
    return head + b"".join(struct.pack("<IQQQ", *l) for l in locs) + b"".join(recs), locs


def patch_nodes(buf: bytes) -> dict:
    """FNDP patch table (rank_forge.cpp:43-102) -> {label: [node_id, ...]}."""
    assert buf[:4] == b"FNDP"
    at = 4 + 2 + 8
    (graphs,) = struct.unpack_from("<I", buf, at)
    at += 4
    out = {}
    for _ in range(graphs):
        label, count = struct.unpack_from("<II", buf, at)
        at += 8
        nodes = []
        for _ in range(count):
            (node,) = struct.unpack_from("<I", buf, at)
            at += 4 + 8
            for _ in range(2):  # stub name, real name
                (n,) = struct.unpack_from("<I", buf, at)
                at += 4 + n
            for _ in range(2):  # rank offsets, world offsets
                (n,) = struct.unpack_from("<I", buf, at)
                at += 4 + 4 * n
            at += 1  # patch_width
            nodes.append(node)
        out[label] = nodes
    assert at == len(buf)
    return out
