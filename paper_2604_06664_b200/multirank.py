"""Multi-GPU orchestration for the LOAD path: one process per GPU.

The graph set is not sharded: every TP rank needs its whole graph set for its
own (rank, world) (reference SPEC.md:474, per-rank PrepareFn pipeline.cpp:504-514).
So N GPUs run N replicas, each materializing its own rank. The one exchange step is a
one-time broadcast of the read-only template store:

* `ipc`  — rank 0 DMAs the store from host into HBM and exports it (CUDA IPC);
           every other rank pulls it GPU->GPU over NVLink (fdy_store_import).
* `host` — every rank DMAs the store from (shared, page-cached) host memory.

torch.distributed is plumbing only: barriers, the handle broadcast and the
max-over-ranks timing reduction. No collective touches the data path.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

TP_WORLD = 8


def tp_rank(global_rank: int, tp_world: int = TP_WORLD) -> int:
    """The TP rank a process materializes: ranks wrap modulo the TP degree."""
    return global_rank % tp_world


@dataclass
class RankGroup:
    """torch.distributed wrapper that degrades to a single process."""

    rank: int = 0
    world: int = 1
    local: int = 0

    @classmethod
    def from_env(cls) -> "RankGroup":
        return cls(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                   int(os.environ.get("LOCAL_RANK", "0")))

    def init(self, backend: str) -> None:
        if self.world > 1:
            import torch.distributed as dist

            if not dist.is_initialized():
                dist.init_process_group(backend, init_method="env://")

    def barrier(self) -> None:
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist

        device = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def broadcast_object(self, obj, src: int = 0):
        if self.world == 1:
            return obj
        import torch.distributed as dist

        box = [obj if self.rank == src else None]
        dist.broadcast_object_list(box, src=src)
        return box[0]

    def close(self) -> None:
        if self.world > 1:
            import torch.distributed as dist

            if dist.is_initialized():
                dist.destroy_process_group()


def distribute_store(group: RankGroup, api, dev, blob: bytes | None, mode: str = "host"):
    """Returns this rank's device-resident copy of the store.

    mode "host": each rank uploads `blob` itself (blob must be given on every rank).
    mode "ipc":  rank 0 uploads and exports; the others import over NVLink.
    """
    if mode == "host" or group.world == 1:
        return api.store_upload(dev, blob)
    if group.rank == 0:
        store = api.store_upload(dev, blob)
        handle = api.store_export(store)
    else:
        store, handle = None, None
    handle = group.broadcast_object(handle, src=0)
    if group.rank != 0:
        store = api.store_import(dev, handle)
    group.barrier()  # every peer has finished pulling before rank 0 may free
    return store
