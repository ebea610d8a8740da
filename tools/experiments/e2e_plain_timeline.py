import os, sys, json, ctypes
sys.path.insert(0, os.getcwd())
from paper_2604_06664_b200 import capi
import paper_2604_06664_b200 as foundry
root = "/tmp/foundry_bench_qwen3-235b-a22b"
plain = root + "/" + os.environ.get("ARCHIVE", "plain")
if not os.path.exists(plain + "/manifest"):  # the bench's archives, or fresh ones
    w = foundry.workload_from_text(open(foundry.workload_path("qwen3-235b-a22b")).read())
    foundry.save(w, root + "/b200")
    foundry.save(w, plain, b200_artifacts=False)
m = json.load(open(plain + "/manifest"))
hdr = capi.store_header(open(root + "/b200/templates.fdt", "rb").read())
api = capi.CApi(); dev = api.device_open(0)
host = api.host_alloc(dev, hdr["members_image_bytes"])
for lanes in [int(x) for x in os.environ.get("LANES", "16").split(",")]:
    for i in range(int(os.environ.get("REPS", "4"))):
        t = api.prepare_archive(dev, plain, 0, 8, m["allocator"]["base"] + 0x10000, lanes, host,
                                hdr["members_image_bytes"])
        print(json.dumps({"lanes": lanes, **{k: round(v, 2) for k, v in t.items() if k.endswith("_ms")}}), flush=True)
