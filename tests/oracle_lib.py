"""ctypes wrapper of oracle/foundry_oracle.c (TEST INFRASTRUCTURE: the checker)."""
from __future__ import annotations

import ctypes
import json
import os


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Oracle:
    def __init__(self, path: str):
        self.lib = ctypes.CDLL(path)
        self.lib.fo_crc64.restype = ctypes.c_uint64
        self.lib.fo_crc64.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
        self.lib.fo_crc64_bitwise.restype = ctypes.c_uint64
        self.lib.fo_crc64_bitwise.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
        self.lib.fo_graph_count.restype = ctypes.c_int64
        self.lib.fo_graph_count.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
        self.lib.fo_materialize_container.restype = ctypes.c_int
        self.lib.fo_materialize_container_ex.restype = ctypes.c_int
        self.lib.fo_free.argtypes = [ctypes.c_void_p]

    def crc64(self, data: bytes) -> int:
        return self.lib.fo_crc64(data, len(data))

    def crc64_bitwise(self, data: bytes) -> int:
        return self.lib.fo_crc64_bitwise(data, len(data))

    def materialize(self, graphs: bytes, patch: bytes, real_hash: int, rank: int, world: int,
                    old_base: int, final_offset: int, new_base: int | None = None,
                    lanes: int = 4, slots: bytes = b"", values=()) -> tuple[bytes, int]:
        out = ctypes.POINTER(ctypes.c_uint8)()
        n = ctypes.c_size_t()
        nr = ctypes.c_uint64()
        err = ctypes.create_string_buffer(512)
        nb = old_base if new_base is None else new_base
        vals = (ctypes.c_uint64 * max(1, len(values)))(*values)
        rc = self.lib.fo_materialize_container_ex(
            graphs, ctypes.c_size_t(len(graphs)), patch, ctypes.c_size_t(len(patch)),
            slots, ctypes.c_size_t(len(slots)), vals, ctypes.c_uint32(len(values)),
            ctypes.c_uint64(real_hash), ctypes.c_uint32(rank), ctypes.c_uint32(world),
            ctypes.c_uint64(old_base), ctypes.c_uint64(final_offset), ctypes.c_uint64(nb),
            ctypes.c_uint(lanes), ctypes.byref(out), ctypes.byref(n), ctypes.byref(nr), err,
            ctypes.c_size_t(512))
        if rc:
            raise OracleError(rc, err.value.decode())
        data = ctypes.string_at(out, n.value)
        self.lib.fo_free(out)
        return data, nr.value

    def materialize_archive(self, archive: str, rank: int, world: int, delta: int = 0,
                            lanes: int = 4, values=()) -> tuple[bytes, int]:
        with open(os.path.join(archive, "manifest")) as f:
            m = json.load(f)
        graphs = open(os.path.join(archive, "graphs.bin"), "rb").read()
        patch = open(os.path.join(archive, "patch.bin"), "rb").read()
        slots = b""
        if "comm_slots.bin" in m["files"]:
            slots = open(os.path.join(archive, "comm_slots.bin"), "rb").read()
        base = m["allocator"]["base"]
        return self.materialize(graphs, patch, m["comm"]["real_binary_hash"], rank, world, base,
                                m["allocator"]["final_offset"], base + delta, lanes, slots, values)
