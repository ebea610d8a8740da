# e2e (C-ABI prepare_archive) timing of the headline archive: median over reps
import os, sys, json, statistics
sys.path.insert(0, os.getcwd())
from paper_2604_06664_b200 import capi
A = "/tmp/foundry_bench_qwen3-235b-a22b/b200"
api = capi.CApi(); dev = api.device_open(0)
h = capi.store_header(open(A + "/templates.fdt", "rb").read())
base = json.load(open(A + "/manifest"))["allocator"]["base"]
out = api.host_alloc(dev, h["members_image_bytes"])
reps = int(os.environ.get("REPS", "4"))
rows = [api.prepare_archive(dev, A, 0, 8, base + 0x10000, 16, out, h["members_image_bytes"]) for _ in range(reps + 1)][1:]
med = {k: round(statistics.median(r[k] for r in rows), 3) for k in ("total_ms", "read_ms", "integrity_ms", "d2h_ms")}
print(os.environ.get("TAG", ""), med, "min total %.3f max %.3f" % (min(r["total_ms"] for r in rows), max(r["total_ms"] for r in rows)), file=sys.stderr)
if len(sys.argv) > 1:
    for f in sorted(os.listdir(A)):
        p = os.path.join(A, f)
        print(f, os.path.getsize(p) if os.path.isfile(p) else sum(os.path.getsize(os.path.join(p, x)) for x in os.listdir(p)), file=sys.stderr)
