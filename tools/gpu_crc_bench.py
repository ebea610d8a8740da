"""GPU CRC-64/XZ throughput (f1): crc_blocks + crc_fold kernel time over the
archive-sized input (3 segments, 277 MB, like the headline archive's files),
cold L2 (inputs larger than L2), checked against the host CRC.

    python tools/gpu_crc_bench.py
"""
from __future__ import annotations

import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_06664_b200 import capi  # noqa: E402


def main() -> None:
    rng = np.random.default_rng(7)
    sizes = [188_300_000, 71_000_000, 18_300_000]
    parts, ranges, off = [], [], 0
    for n in sizes:
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        parts.append(b + b"\0" * ((-n) % 256))
        ranges.append((off, n))
        off += len(parts[-1])
    data = b"".join(parts)
    api = capi.CApi()
    dev = api.device_open(0)
    ms = []
    for _ in range(6):
        dig, k = api.crc64(dev, data, ranges)
        ms.append(k)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from oracle_lib import Oracle
    orc = Oracle(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_build",
                              "liboracle.so"))
    ok = dig == [orc.crc64(p[:n]) for p, n in zip(parts, sizes)]
    total = sum(sizes)
    med = statistics.median(ms[1:])
    print(json.dumps({"bytes": total, "kernel_ms_median": med, "kernel_ms_best": min(ms[1:]),
                      "GBps": total / (med * 1e-3) / 1e9, "matches_oracle": ok}))


if __name__ == "__main__":
    main()
