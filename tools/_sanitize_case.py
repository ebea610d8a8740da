"""Small end-to-end case for compute-sanitizer: SAVE a small moe archive, run the
fused materialize kernel (with and without relocation) and the GPU CRC through
the C-ABI, LOAD + replay + device-updates serve through the Python API."""
import json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_06664_b200 as foundry
from paper_2604_06664_b200 import capi

t = tempfile.mkdtemp()
spec = foundry.preset("moe-spmd"); spec.batch_max = 24; spec.thresholds = [5, 9, 17]
foundry.save(spec, t + "/a")
blob = open(t + "/a/templates.fdt", "rb").read()
base = json.load(open(t + "/a/manifest"))["allocator"]["base"]
api = capi.CApi(); dev = api.device_open(0)
store = api.store_upload(dev, blob)
m, _ = api.materialize(dev, store, 1, 4, 0)
api.materialize(dev, store, 1, 4, base + 0x10000, m)
api.crc64(dev, blob, [(0, len(blob)), (0, 7), (16, 65536 * 3 + 5)])
api.lib.fdy_members_free(m); api.lib.fdy_store_free(store); api.lib.fdy_device_close(dev)
h = foundry.load(t + "/a", rank=1, world=4, device_updates=True)
for b in h.batches()[:6]:
    h.serve(b); h.replay(b)
h.close()
print("sanitize case ok")
