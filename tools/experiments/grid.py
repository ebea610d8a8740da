"""Grid-size sweep of the fused materialize launch (headline archive, cold L2)."""
import ctypes, json, os, statistics, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2604_06664_b200 import capi
A = "/tmp/foundry_bench_qwen3-235b-a22b/b200"
blob = open(A + "/templates.fdt", "rb").read()
base = json.load(open(A + "/manifest"))["allocator"]["base"]
api = capi.CApi(); dev = api.device_open(0); store = api.store_upload(dev, blob)
members, _ = api.materialize(dev, store, 0, 8, base + 0x10000)
fw = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); fr = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
for grid in [int(g) for g in (sys.argv[1].split(",") if len(sys.argv) > 1 else "148,296,444,592,740,888,1036".split(","))]:
    ts = []
    for i in range(15):
        fw.zero_(); torch.count_nonzero(fr); torch.cuda.synchronize()
        desc = capi.MaterializeDesc(0, 8, base + 0x10000, None, 0, grid)
        ms = ctypes.c_float()
        api.check(api.lib.fdy_materialize_into(dev, store, ctypes.byref(desc), members, ctypes.byref(ms)))
        if i >= 3: ts.append(ms.value * 1e3)
    print(grid, round(statistics.median(ts), 2), round(min(ts), 2))
