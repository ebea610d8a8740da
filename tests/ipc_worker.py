"""Worker of the multi-process fan-out tests in test_gpu_capi.py (one process
per rank, all on cuda:0; gloo carries the exported handles).

    RANK=r WORLD_SIZE=n MASTER_ADDR=127.0.0.1 MASTER_PORT=p python ipc_worker.py <archive> <outdir> [ipc|chain]
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    arch, outdir = sys.argv[1], sys.argv[2]
    mode = sys.argv[3] if len(sys.argv) > 3 else "ipc"
    import paper_2604_06664_b200 as foundry
    from paper_2604_06664_b200 import capi
    from paper_2604_06664_b200.multirank import RankGroup, distribute_store

    g = RankGroup.from_env()
    g.init("gloo")
    api = capi.CApi()
    dev = api.device_open(0)
    blob = open(os.path.join(arch, "templates.fdt"), "rb").read() if g.rank == 0 else None
    store = distribute_store(g, api, dev, blob, mode)
    base = json.load(open(os.path.join(arch, "manifest")))["allocator"]["base"]
    tp = 2 + g.rank
    members, _ = api.materialize(dev, store, tp, 8, base + 0x10000 * (g.rank + 1))
    arena = api.members_download(members)
    with open(os.path.join(outdir, "rank%d.fndg" % g.rank), "wb") as f:
        f.write(foundry._foundry._decode_member_images(arch, arena))
    api.lib.fdy_members_free(members)
    g.barrier()  # the exporter keeps its store alive until every importer is done
    api.lib.fdy_store_free(store)
    api.lib.fdy_device_close(dev)
    g.close()


if __name__ == "__main__":
    main()
