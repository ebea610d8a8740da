"""Worker of test_gpu_capi.py::test_forged_store_is_rejected_or_contained: byte
flips in templates.fdt with the manifest digest made consistent again, so only
the store's own validation stands between a forged file and the device. Every
mutation must either materialize (fdy_prepare_archive, then a LOAD + replay of
two batches) or fail with a FoundryError that is not a CUDA error; a fault on
the device would poison the context, so the worker runs in its own process.

    python store_fuzz_worker.py <archive> <scratch> <seed> <n>
Prints one JSON line {"ok": n_ok, "rejected": n_rejected, "messages": [...]}.
"""
from __future__ import annotations

import json
import os
import random
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

STICKY = ("ILLEGAL_ADDRESS", "illegal memory access", "MISALIGNED", "misaligned", "LAUNCH_FAILED",
          "launch failure", "ILLEGAL_INSTRUCTION", "HARDWARE_STACK_ERROR", "unspecified launch failure")


def main() -> None:
    src, scratch, seed, n = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    import paper_2604_06664_b200 as foundry
    from paper_2604_06664_b200 import capi

    api = capi.CApi()
    dev = api.device_open(0)
    blob = open(os.path.join(src, "templates.fdt"), "rb").read()
    hdr = capi.store_header(blob)
    host = api.host_alloc(dev, hdr["members_image_bytes"] + 4096)
    r = random.Random(seed)
    ok = rejected = 0
    messages = set()
    for i in range(n):
        arch = os.path.join(scratch, "f%d" % i)
        shutil.copytree(src, arch)
        b = bytearray(blob)
        # half the flips land in the header and tables (the first 64 KiB hold
        # the header and, for a small store, most tables), half anywhere
        for _ in range(r.choice([1, 2, 4])):
            at = r.randrange(min(len(b), 65536)) if r.random() < 0.5 else r.randrange(len(b))
            b[at] ^= r.randrange(1, 256)
        open(os.path.join(arch, "templates.fdt"), "wb").write(bytes(b))
        m = json.load(open(os.path.join(arch, "manifest")))
        m["files"]["templates.fdt"] = foundry._foundry._crc64(bytes(b))
        json.dump(m, open(os.path.join(arch, "manifest"), "w"))
        try:
            api.prepare_archive(dev, arch, 1, 2, 0, 2, host, hdr["members_image_bytes"] + 4096)
            h = foundry.load(arch, rank=1, world=2)
            try:  # a handle left to the garbage collector would keep the VA range reserved
                for batch in h.batches()[:2]:
                    h.replay(batch)
            finally:
                h.close()
            ok += 1
        except (foundry.FoundryError, capi.CApiError) as e:
            msg = str(e)
            # a driver that refuses a forged launch configuration is a clean
            # error; a fault on the device (sticky, context lost) is not
            assert not any(k in msg for k in STICKY), (i, msg)
            assert "out-of-region" not in msg, (i, msg)  # an earlier handle still holds the range
            rejected += 1
            messages.add(msg.split(":")[0] + ": " + msg.split(":")[-1].strip()[:60])
        shutil.rmtree(arch)
    # the context is still healthy: the untouched archive materializes and replays
    api.prepare_archive(dev, src, 1, 2, 0, 2, host, hdr["members_image_bytes"] + 4096)
    h = foundry.load(src, rank=1, world=2)
    h.replay(h.batches()[0])
    h.close()
    api.lib.fdy_device_close(dev)
    print(json.dumps({"ok": ok, "rejected": rejected, "messages": sorted(messages)[:20]}))


if __name__ == "__main__":
    main()
