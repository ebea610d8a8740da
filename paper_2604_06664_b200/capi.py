"""ctypes binding of the C-ABI (include/foundry_b200.h).

This is the binding a foreign host would write (INTEGRATION.md shows the same
for cgo / JNI); bench.py uses it to drive the kernel layer directly.
"""
from __future__ import annotations

import ctypes
import os
import re
import struct

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfoundry_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "foundry_b200.h")


class MaterializeDesc(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_uint32),
        ("world", ctypes.c_uint32),
        ("new_base", ctypes.c_uint64),
        ("values", ctypes.POINTER(ctypes.c_uint64)),
        ("n_values", ctypes.c_uint32),
        ("grid", ctypes.c_int32),
    ]


class LoadOptions(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_uint32),
        ("world", ctypes.c_uint32),
        ("preallocate", ctypes.c_int32),
        ("prepare_lanes", ctypes.c_uint32),
        ("device", ctypes.c_int32),
        ("relocate", ctypes.c_int32),
        ("skip_binary_restore", ctypes.c_int32),
        ("skip_device_init", ctypes.c_int32),
        ("base_shift_granules", ctypes.c_int64),
        ("extra_prewindow_alloc", ctypes.c_int32),
        ("share_execs", ctypes.c_int32),
        ("device_updates", ctypes.c_int32),
        ("comm_values", ctypes.POINTER(ctypes.c_uint64)),
        ("n_comm_values", ctypes.c_uint32),
    ]


class PrepareTimings(ctypes.Structure):
    _fields_ = [
        ("total_ms", ctypes.c_double),
        ("read_ms", ctypes.c_double),
        ("integrity_ms", ctypes.c_double),
        ("materialize_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("crc_kernel_ms", ctypes.c_float),
        ("kernel_ms", ctypes.c_float),
        ("h2d_bytes", ctypes.c_uint64),
        ("d2h_bytes", ctypes.c_uint64),
        ("member_bytes", ctypes.c_uint64),
        ("graphs", ctypes.c_uint64),
        ("nodes", ctypes.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class CApiError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def declared_functions(header: str = HEADER) -> list[str]:
    """Every fdy_* function the public header declares."""
    text = open(header).read()
    return sorted(set(re.findall(r"\b(fdy_[a-z0-9_]+)\s*\(", text)))


class CApi:
    def __init__(self, path: str = LIB_PATH):
        self.lib = ctypes.CDLL(path)
        L = self.lib
        P = ctypes.c_void_p
        L.fdy_last_error.restype = ctypes.c_char_p
        L.fdy_version.restype = ctypes.c_char_p
        L.fdy_device_count.restype = ctypes.c_int
        L.fdy_device_open.argtypes = [ctypes.c_int, ctypes.POINTER(P)]
        L.fdy_device_close.argtypes = [P]
        L.fdy_sync.argtypes = [P]
        L.fdy_store_upload.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(P)]
        L.fdy_store_fanout.argtypes = [P, P, ctypes.POINTER(P)]
        L.fdy_store_free.argtypes = [P]
        L.fdy_store_export.argtypes = [P, ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint64)]
        L.fdy_store_import.argtypes = [P, ctypes.c_char_p, ctypes.c_uint64, ctypes.POINTER(P)]
        L.fdy_store_fanout_chain.argtypes = [P, ctypes.POINTER(P), ctypes.c_uint32, ctypes.c_uint64,
                                             ctypes.POINTER(P)]
        L.fdy_chain_create.argtypes = [P, ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(P), ctypes.c_char_p]
        L.fdy_chain_seed.argtypes = [P, ctypes.c_void_p]
        L.fdy_chain_pull.argtypes = [P, ctypes.c_char_p]
        L.fdy_chain_finish.argtypes = [P, ctypes.POINTER(P)]
        L.fdy_chain_free.argtypes = [P]
        L.fdy_store_members_bytes.argtypes = [P]
        L.fdy_store_members_bytes.restype = ctypes.c_size_t
        L.fdy_materialize.argtypes = [P, P, ctypes.POINTER(MaterializeDesc), ctypes.POINTER(P),
                                      ctypes.POINTER(ctypes.c_float)]
        L.fdy_materialize_into.argtypes = [P, P, ctypes.POINTER(MaterializeDesc), P,
                                           ctypes.POINTER(ctypes.c_float)]
        L.fdy_members_write_probe.argtypes = [P, ctypes.POINTER(ctypes.c_float)]
        L.fdy_members_bytes.argtypes = [P]
        L.fdy_members_bytes.restype = ctypes.c_size_t
        L.fdy_members_download.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t]
        L.fdy_members_free.argtypes = [P]
        L.fdy_materialize_timed_split.argtypes = [P, P, ctypes.POINTER(MaterializeDesc), P,
                                                  ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]
        L.fdy_crc64_segments.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t,
                                         ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.POINTER(ctypes.c_float)]
        L.fdy_prepare_archive.argtypes = [P, ctypes.c_char_p, ctypes.POINTER(MaterializeDesc),
                                          ctypes.c_uint32, ctypes.c_void_p, ctypes.c_size_t,
                                          ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(PrepareTimings)]
        L.fdy_host_alloc.argtypes = [P, ctypes.c_size_t]
        L.fdy_host_alloc.restype = ctypes.c_void_p
        L.fdy_host_free.argtypes = [ctypes.c_void_p]
        L.fdy_load_options_init.argtypes = [ctypes.POINTER(LoadOptions)]
        L.fdy_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(LoadOptions), ctypes.POINTER(P)]
        L.fdy_serving_replay.argtypes = [P, ctypes.c_uint32, ctypes.c_char_p, ctypes.c_size_t,
                                         ctypes.POINTER(ctypes.c_size_t)]
        L.fdy_serving_close.argtypes = [P]
        L.fdy_serving_capture_graph.argtypes = [P, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_size_t,
                                                ctypes.POINTER(ctypes.c_size_t)]

    def check(self, rc: int) -> None:
        if rc:
            raise CApiError(rc, self.lib.fdy_last_error().decode(errors="backslashreplace"))

    # ---- session layer (the reference's LOAD surface)
    def load(self, archive: str, rank: int = 0, world: int = 1, relocate: bool = False,
             share_execs: bool = False, comm_values=()):
        o = LoadOptions()
        self.lib.fdy_load_options_init(ctypes.byref(o))
        o.rank, o.world, o.relocate, o.share_execs = rank, world, int(relocate), int(share_execs)
        vals = (ctypes.c_uint64 * max(1, len(comm_values)))(*comm_values)
        o.comm_values, o.n_comm_values = vals, len(comm_values)
        h = ctypes.c_void_p()
        self.check(self.lib.fdy_load(archive.encode(), ctypes.byref(o), ctypes.byref(h)))
        return h

    def serving_replay(self, h, batch: int) -> str:
        n = ctypes.c_size_t()
        self.check(self.lib.fdy_serving_replay(h, batch, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        self.check(self.lib.fdy_serving_replay(h, batch, buf, n.value + 1, ctypes.byref(n)))
        return buf.raw[:n.value].decode()

    def serving_capture_graph(self, h, batch: int) -> bytes:
        n = ctypes.c_size_t()
        self.check(self.lib.fdy_serving_capture_graph(h, batch, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        self.check(self.lib.fdy_serving_capture_graph(h, batch, buf, n.value, ctypes.byref(n)))
        return buf.raw[:n.value]

    # ---- kernel layer
    def device_open(self, ordinal: int = 0):
        h = ctypes.c_void_p()
        self.check(self.lib.fdy_device_open(ordinal, ctypes.byref(h)))
        return h

    def store_upload(self, dev, blob: bytes):
        h = ctypes.c_void_p()
        self.check(self.lib.fdy_store_upload(dev, blob, len(blob), ctypes.byref(h)))
        return h

    def store_export(self, store) -> tuple[bytes, int]:
        handle = ctypes.create_string_buffer(64)
        n = ctypes.c_uint64()
        self.check(self.lib.fdy_store_export(store, handle, ctypes.byref(n)))
        return handle.raw, n.value

    def store_import(self, dev, exported: tuple[bytes, int]):
        handle, nbytes = exported
        h = ctypes.c_void_p()
        self.check(self.lib.fdy_store_import(dev, handle, nbytes, ctypes.byref(h)))
        return h

    def store_fanout_chain(self, src, devs, chunk_bytes: int = 0) -> list:
        """In-process pipelined chain: devs[0] pulls from src, devs[i] from devs[i-1]."""
        n = len(devs)
        arr = (ctypes.c_void_p * n)(*[d.value if isinstance(d, ctypes.c_void_p) else d for d in devs])
        outs = (ctypes.c_void_p * n)()
        self.check(self.lib.fdy_store_fanout_chain(src, arr, n, chunk_bytes, outs))
        return [ctypes.c_void_p(o) for o in outs]

    def chain_create(self, dev, nbytes: int, chunk_bytes: int = 0):
        h = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        self.check(self.lib.fdy_chain_create(dev, nbytes, chunk_bytes, ctypes.byref(h), handle))
        return h, handle.raw

    def chain_seed(self, chain, blob: bytes) -> None:
        self.check(self.lib.fdy_chain_seed(chain, blob))

    def chain_pull(self, chain, upstream: bytes) -> None:
        self.check(self.lib.fdy_chain_pull(chain, upstream))

    def chain_finish(self, chain):
        h = ctypes.c_void_p()
        self.check(self.lib.fdy_chain_finish(chain, ctypes.byref(h)))
        self.lib.fdy_chain_free(chain)
        return h

    @staticmethod
    def _desc(rank: int, world: int, new_base: int, values=()):
        desc = MaterializeDesc(rank, world, new_base, None, 0, 0)
        if values:
            arr = (ctypes.c_uint64 * len(values))(*values)
            desc.values = arr
            desc.n_values = len(values)
            desc._keep = arr  # the table must outlive the call
        return desc

    def materialize(self, dev, store, rank: int, world: int, new_base: int = 0, members=None,
                    values=()):
        desc = self._desc(rank, world, new_base, values)
        ms = ctypes.c_float()
        if members is None:
            members = ctypes.c_void_p()
            self.check(self.lib.fdy_materialize(dev, store, ctypes.byref(desc), ctypes.byref(members),
                                                ctypes.byref(ms)))
        else:
            self.check(self.lib.fdy_materialize_into(dev, store, ctypes.byref(desc), members,
                                                     ctypes.byref(ms)))
        return members, ms.value

    def materialize_split(self, dev, store, rank: int, world: int, new_base: int, members, values=()):
        """(relocation ms, member-pass ms): the two grids timed apart."""
        desc = self._desc(rank, world, new_base, values)
        r, m = ctypes.c_float(), ctypes.c_float()
        self.check(self.lib.fdy_materialize_timed_split(dev, store, ctypes.byref(desc), members,
                                                        ctypes.byref(r), ctypes.byref(m)))
        return r.value, m.value

    def prepare_archive(self, dev, archive: str, rank: int, world: int, new_base: int = 0,
                        lanes: int = 0, host_out=None, cap: int = 0, values=()) -> dict:
        """The materialization path in one C-ABI call (fdy_prepare_archive)."""
        desc = self._desc(rank, world, new_base, values)
        n = ctypes.c_size_t()
        t = PrepareTimings()
        self.check(self.lib.fdy_prepare_archive(dev, archive.encode(), ctypes.byref(desc),
                                                lanes or (os.cpu_count() or 4), host_out, cap,
                                                ctypes.byref(n), ctypes.byref(t)))
        return t.as_dict()

    def host_alloc(self, dev, nbytes: int):
        p = self.lib.fdy_host_alloc(dev, nbytes)
        if not p:
            raise CApiError(1, self.lib.fdy_last_error().decode(errors="backslashreplace"))
        return p

    def members_download(self, members) -> bytes:
        n = self.lib.fdy_members_bytes(members)
        buf = ctypes.create_string_buffer(n)
        self.check(self.lib.fdy_members_download(members, buf, 0, n))
        return buf.raw

    def crc64(self, dev, data: bytes, ranges):
        n = len(ranges)
        offs = (ctypes.c_uint64 * n)(*[r[0] for r in ranges])
        lens = (ctypes.c_uint64 * n)(*[r[1] for r in ranges])
        out = (ctypes.c_uint64 * n)()
        ms = ctypes.c_float()
        self.check(self.lib.fdy_crc64_segments(dev, data, len(data), offs, lens, n, out, ctypes.byref(ms)))
        return list(out), ms.value


# ---- FNDT store header (foundry/store_format.h) -----------------------------

SECTIONS = ["groups", "timages", "cmeta", "members", "tiles", "didx", "ddata", "rops",
            "kernels", "nodeattrs", "edges", "strings"]


def store_header(blob: bytes) -> dict:
    (magic, version, flags, header_bytes, n_groups, n_members, n_kernels, n_tiles, tile_chunks,
     n_diffs, n_rank_ops) = struct.unpack_from("<4sHHIIIIIIII", blob, 0)
    assert magic == b"FNDT", "not a template store"
    u64 = struct.unpack_from("<7Q", blob, 40)
    n_plain, n_values, slots_crc = struct.unpack_from("<IIQ", blob, 96)
    secs = struct.unpack_from("<%dQ" % (2 * len(SECTIONS)), blob, 112)
    return {
        "version": version, "n_groups": n_groups, "n_members": n_members, "n_kernels": n_kernels,
        "n_tiles": n_tiles, "tile_chunks": tile_chunks, "n_diffs": n_diffs, "n_rank_ops": n_rank_ops,
        "source_graphs_crc": u64[0], "source_patch_crc": u64[1], "old_base": u64[2],
        "final_offset": u64[3], "real_comm_hash": u64[4], "members_image_bytes": u64[5],
        "total_nodes": u64[6], "n_plain_tiles": n_plain, "n_values": n_values,
        "source_slots_crc": slots_crc,
        "sec": {n: (secs[2 * i], secs[2 * i + 1]) for i, n in enumerate(SECTIONS)},
    }


def algorithmic_bytes(h: dict) -> dict:
    """Compulsory HBM traffic of one fused K2+K1+K3 launch:
    templates + chunk meta read once, every diff / rank op / tile read once,
    every member image written once. `member_pass` is the fdy_materialize_kernel
    grid's own share (it reads the relocated templates, not the chunk meta)."""
    s = h["sec"]
    read = (s["timages"][1] + s["cmeta"][1] + s["didx"][1] + s["ddata"][1]
            + s["rops"][1] + s["tiles"][1])
    write = h["members_image_bytes"]
    return {"read": read, "write": write, "total": read + write,
            "member_pass": read - s["cmeta"][1] + write}
