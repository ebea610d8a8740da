"""Comm-slot tables for tests (TEST INFRASTRUCTURE).

The stub layer authors which argument bytes of a comm stub hold per-rank
deployment state (archive.hpp CommSlot; stub layout rank@0 world@8 buf@16
payload@24, reference rank_forge.cpp:18-22). Two tables over every patched
comm node of an archive:

* `stress`: writes that straddle 16-byte chunks (offset 12, 8 bytes), overlap
  the rank/world bytes (table order: slots win), 4- and 1-byte widths, and a
  value index that cycles through the table;
* `deploy`: what a deployment writes — a peer buffer address at buf@16 and a
  communicator handle over payload@24 — so replays stay valid when the peer
  buffer values are mapped addresses.
"""
from __future__ import annotations

import os

import fndg

N_VALUES = 6


def stress_table(archive: str) -> dict:
    nodes = fndg.patch_nodes(open(os.path.join(archive, "patch.bin"), "rb").read())
    out = {}
    for label, ids in nodes.items():
        slots = []
        for k, n in enumerate(ids):
            slots.append((n, 12, (k + label) % N_VALUES, 8))  # straddles chunks 0|1, overlaps world@8
            slots.append((n, 28, (k + 1) % N_VALUES, 4))
            slots.append((n, 5, (k + 2) % N_VALUES, 1))        # inside rank@0
        out[label] = slots
    return out


def deploy_table(archive: str) -> dict:
    nodes = fndg.patch_nodes(open(os.path.join(archive, "patch.bin"), "rb").read())
    return {label: [slot for k, n in enumerate(ids)
                    for slot in ((n, 16, 1 + k % (N_VALUES - 1), 8), (n, 24, 0, 8))]
            for label, ids in nodes.items()}


def rank_values(rank: int, base: int = 0) -> list:
    """A distinct table per rank: a comm handle, then peer buffer addresses
    (granule-aligned offsets from `base` when given, so they are mapped)."""
    handle = 0xC0DE000000000000 | (rank << 32) | 0xA5A5
    if base:
        return [handle] + [base + 0x10000 * (1 + (rank * 7 + i) % 64) for i in range(N_VALUES - 1)]
    return [handle] + [0x7F0000000000 + (rank << 24) + 0x100 * i + 0x11 for i in range(N_VALUES - 1)]
