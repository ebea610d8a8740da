"""Worker of test_gpu_capi.py::test_chain_link_times_out_on_a_silent_predecessor:
rank 0 creates a chain link and never seeds it; rank r > 0 pulls from rank
r - 1 with a short timeout, and every one of them must get the timeout error
from fdy_chain_finish (a link that gave up does not forward).

    RANK=r WORLD_SIZE=n MASTER_ADDR=127.0.0.1 MASTER_PORT=p python chain_timeout_worker.py
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    from paper_2604_06664_b200 import capi
    from paper_2604_06664_b200.multirank import RankGroup

    g = RankGroup.from_env()
    g.init("gloo")
    api = capi.CApi()
    dev = api.device_open(0)
    chain, handle = api.chain_create(dev, 1 << 20)
    handles = g.all_gather_object(handle)
    rc = 0
    if g.rank > 0:
        os.environ["FOUNDRY_CHAIN_TIMEOUT_MS"] = "1500"
        api.chain_pull(chain, handles[g.rank - 1])
        try:
            api.chain_finish(chain)
            rc = 3  # should have timed out
        except capi.CApiError as e:
            rc = 0 if "no progress" in str(e) else 4
    g.barrier()  # every link stays alive until its successor is done
    if g.rank == 0:
        api.lib.fdy_chain_free(chain)
    api.lib.fdy_device_close(dev)
    g.close()
    return rc


if __name__ == "__main__":
    sys.exit(main())
