import os, sys, json
sys.path.insert(0, os.getcwd())
from paper_2604_06664_b200 import capi
A="/tmp/foundry_bench_qwen3-235b-a22b/b200"
api=capi.CApi(); dev=api.device_open(0)
h=capi.store_header(open(A+"/templates.fdt","rb").read())
base=json.load(open(A+"/manifest"))["allocator"]["base"]
out=api.host_alloc(dev,h["members_image_bytes"])
for i in range(4):
    t=api.prepare_archive(dev,A,0,8,base+0x10000,16,out,h["members_image_bytes"])
    print({k:round(v,3) for k,v in t.items() if k.endswith("_ms")}, file=sys.stderr)
