import os, sys, json, ctypes
sys.path.insert(0, os.getcwd())
from paper_2604_06664_b200 import capi
import paper_2604_06664_b200 as foundry
root = "/tmp/foundry_bench_qwen3-235b-a22b"
plain = root + "/plain"
m = json.load(open(plain + "/manifest"))
hdr = capi.store_header(open(root + "/b200/templates.fdt", "rb").read())
api = capi.CApi(); dev = api.device_open(0)
host = api.host_alloc(dev, hdr["members_image_bytes"])
for i in range(4):
    t = api.prepare_archive(dev, plain, 0, 8, m["allocator"]["base"] + 0x10000, 16, host, hdr["members_image_bytes"])
    print(json.dumps({k: round(v, 2) for k, v in t.items() if k.endswith("_ms")}), flush=True)
