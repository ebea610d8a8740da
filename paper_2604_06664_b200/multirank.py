"""Multi-GPU orchestration for the LOAD path: one process per GPU.

The graph set is not sharded: every TP rank needs its whole graph set for its
own (rank, world) (reference SPEC.md:474, per-rank PrepareFn pipeline.cpp:504-514).
So N GPUs run N replicas, each materializing its own rank. The one exchange step is a
one-time broadcast of the read-only template store:

* `ipc`  — rank 0 DMAs the store from host into HBM and exports it (CUDA IPC);
           every other rank pulls it GPU->GPU over NVLink (fdy_store_import).
* `host` — every rank DMAs the store from (shared, page-cached) host memory.
* `chain` — pipelined chain over the ranks of a node (SURVEY §8e ii): local
           rank 0 seeds its copy from host memory chunk by chunk, rank r pulls
           each chunk from rank r-1 as soon as it landed there (fdy_chain_*:
           a progress word in HBM polled by the GPU), so the store crosses
           every NVLink hop once, pipelined, instead of rank 0's egress
           carrying N-1 copies.

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

    def all_gather_object(self, obj) -> list:
        if self.world == 1:
            return [obj]
        import torch.distributed as dist

        out = [None] * self.world
        dist.all_gather_object(out, obj)
        return out

    def close(self) -> None:
        if self.world > 1:
            import torch.distributed as dist

            if dist.is_initialized():
                dist.destroy_process_group()


def node_leader(group: RankGroup) -> int:
    """Global rank of the first process on this rank's node (torchrun numbers
    ranks node by node, so it is global rank - local rank)."""
    return group.rank - group.local


def distribute_store(group: RankGroup, api, dev, blob: bytes | None, mode: str = "host"):
    """Returns this rank's device-resident copy of the store.

    mode "host": each rank uploads `blob` itself (blob must be given on every rank).
    mode "ipc":  local rank 0 of every node uploads and exports; the other ranks of
                 that node import it over NVLink (CUDA IPC handles are node-local).
    mode "chain": local rank 0 of every node seeds a pipelined chain through the
                 node's ranks in global-rank order (blob needed on local rank 0).
    """
    if mode == "host" or group.world == 1:
        return api.store_upload(dev, blob)
    if mode == "chain":
        return _chain(group, api, dev, blob)
    leader = node_leader(group)
    if group.rank == leader:
        store = api.store_upload(dev, blob)
        handle = api.store_export(store)
    else:
        store, handle = None, None
    handles = group.all_gather_object((leader, handle) if group.rank == leader else None)
    if group.rank != leader:
        mine = [h for h in handles if h is not None and h[0] == leader]
        if not mine:  # no exporter on this node: fall back to a host upload
            store = api.store_upload(dev, blob)
        else:
            store = api.store_import(dev, mine[0][1])
    group.barrier()  # every peer has finished pulling before a leader may free
    return store


def _chain(group: RankGroup, api, dev, blob: bytes | None):
    """mode "chain": the node's ranks in global-rank order form the chain; the
    node leader is its head. Every rank needs the store's size (blob or the
    leader's broadcast)."""
    leader = node_leader(group)
    size = group.all_gather_object(len(blob) if group.rank == leader else None)[leader]
    chain, handle = api.chain_create(dev, size)
    links = group.all_gather_object((leader, group.rank, handle))
    if group.rank == leader:
        api.chain_seed(chain, blob)
    else:
        upstream = [h for (l, r, h) in links if l == leader and r == group.rank - 1]
        assert upstream, "chain fan-out: no predecessor on this node"
        api.chain_pull(chain, upstream[0])
    store = api.chain_finish(chain)
    group.barrier()  # every link has finished reading its predecessor
    return store

