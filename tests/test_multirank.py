"""N>1 host logic on CPU: two gloo processes run the bench orchestration
(rank 0 writes the archive, barrier, each process materializes its own TP rank,
max-over-ranks reduction, object broadcast of the store handle). The kernel is
replaced by its NumPy emulation; each rank's graph set must equal the oracle's
for that rank."""
from __future__ import annotations

import os
import socket
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank: int, world: int, port: int, workdir: str, queue) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    try:
        import json

        import store_emulator as emu
        from oracle_lib import Oracle
        import paper_2604_06664_b200 as foundry
        from paper_2604_06664_b200.multirank import RankGroup, TP_WORLD, tp_rank

        g = RankGroup.from_env()
        g.init("gloo")
        arch = os.path.join(workdir, "moe")
        if g.rank == 0:
            spec = foundry.preset("moe-spmd")
            spec.batch_max = 24
            spec.thresholds = [5, 9, 17]
            foundry.save(spec, arch)
        g.barrier()
        # the store bytes travel once from rank 0 (the handle/object broadcast path)
        blob = open(os.path.join(arch, "templates.fdt"), "rb").read() if g.rank == 0 else None
        blob = g.broadcast_object(blob, src=0)
        r = tp_rank(g.rank + 5)  # ranks 5 and 6 of the TP-8 group
        m = json.load(open(os.path.join(arch, "manifest")))
        delta = 0x10000 * (g.rank + 1)
        arena = emu.expand(blob, r, TP_WORLD, m["allocator"]["base"] + delta)
        got = foundry._foundry._decode_member_images(arch, arena)
        want, _ = Oracle(os.path.join(ROOT, "oracle", "_build", "liboracle.so")).materialize_archive(
            arch, r, TP_WORLD, delta)
        worst = g.max(float(g.rank + 1))
        queue.put((g.rank, got == want, worst, r))
        g.close()
    except Exception as exc:  # surface worker failures to the parent
        queue.put((rank, repr(exc), None, None))


def test_two_rank_orchestration_over_gloo(tmp_path, native_build):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(tmp_path), q)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in results] == [True, True], results
    assert all(r[2] == 2.0 for r in results)  # max over ranks
    assert [r[3] for r in results] == [5, 6]


def test_tp_rank_mapping():
    from paper_2604_06664_b200.multirank import tp_rank

    assert [tp_rank(r) for r in range(10)] == [0, 1, 2, 3, 4, 5, 6, 7, 0, 1]


class _FakeApi:
    """Records the store calls distribute_store makes (no GPU)."""

    def __init__(self, rank):
        self.rank, self.calls = rank, []

    def store_upload(self, dev, blob):
        self.calls.append(("upload", len(blob)))
        return ("store", self.rank)

    def store_export(self, store):
        self.calls.append(("export",))
        return "handle-of-%d" % self.rank

    def store_import(self, dev, handle):
        self.calls.append(("import", handle))
        return ("imported", handle)


def _fanout_worker(rank: int, world: int, local: int, port: int, queue) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(local))
    sys.path.insert(0, ROOT)
    try:
        from paper_2604_06664_b200.multirank import RankGroup, distribute_store

        g = RankGroup.from_env()
        g.init("gloo")
        api = _FakeApi(rank)
        distribute_store(g, api, None, b"x" * 64, "ipc")
        queue.put((rank, api.calls))
        g.close()
    except Exception as exc:
        queue.put((rank, repr(exc)))


def test_ipc_fanout_has_one_exporter_per_node():
    """Two 'nodes' of two ranks each (world 4, local ranks 0,1,0,1): each node's
    local rank 0 uploads and exports; its peer imports that node's handle
    (CUDA IPC handles do not cross nodes)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fanout_worker, args=(r, 4, r % 2, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert got[0] == [("upload", 64), ("export",)], got
    assert got[2] == [("upload", 64), ("export",)], got
    assert got[1] == [("import", "handle-of-0")], got
    assert got[3] == [("import", "handle-of-2")], got


class _FileChainApi:
    """Stand-in for the chain C-ABI (fdy_chain_*) with files as links: a
    link's 'HBM' is a file named after its handle; pull waits for the
    predecessor's file. Exercises the orchestration only (who seeds, who pulls
    from whom, across two nodes)."""

    def __init__(self, workdir: str, rank: int):
        self.dir, self.rank = workdir, rank

    def chain_create(self, dev, nbytes, chunk_bytes=0):
        return {"size": nbytes, "path": os.path.join(self.dir, "link%d" % self.rank)}, b"link%d" % self.rank

    def chain_seed(self, chain, blob):
        assert len(blob) == chain["size"]
        open(chain["path"], "wb").write(blob)

    def chain_pull(self, chain, upstream):
        import time
        src = os.path.join(self.dir, upstream.decode())
        for _ in range(6000):
            if os.path.exists(src) and os.path.getsize(src) == chain["size"]:
                break
            time.sleep(0.01)
        data = open(src, "rb").read()
        chain["pulled_from"] = upstream.decode()
        open(chain["path"], "wb").write(data)

    def chain_finish(self, chain):
        return (open(chain["path"], "rb").read(), chain.get("pulled_from"))


def _chain_worker(rank: int, world: int, local: int, port: int, workdir: str, queue) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(local))
    sys.path.insert(0, ROOT)
    try:
        from paper_2604_06664_b200.multirank import RankGroup, distribute_store

        g = RankGroup.from_env()
        g.init("gloo")
        blob = bytes(range(256)) * 1000 if local == 0 else None
        data, pulled_from = distribute_store(g, _FileChainApi(workdir, rank), None, blob, "chain")
        queue.put((rank, data == bytes(range(256)) * 1000, pulled_from))
        g.close()
    except Exception as exc:
        queue.put((rank, repr(exc), None))


def test_chain_fanout_orchestration_over_gloo(tmp_path, native_build):
    """Four processes on two 'nodes' (local ranks 0,1,2 and 0): each node's
    leader seeds its own chain, every other rank pulls from the rank before it
    on its node, and every rank ends with the store's bytes."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    locals_ = [0, 1, 2, 0]
    procs = [ctx.Process(target=_chain_worker, args=(r, 4, locals_[r], port, str(tmp_path), q)) for r in range(4)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in results] == [True] * 4, results
    assert [r[2] for r in results] == [None, "link0", "link1", None]
