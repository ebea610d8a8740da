"""Small end-to-end case for compute-sanitizer: SAVE a small moe archive, run the
fused materialize kernel (with and without relocation) and the GPU CRC through
the C-ABI, LOAD + replay + device-updates serve through the Python API; the
GPU packer on the same archive written without B200 artefacts (store bytes
checked against the offline packer) and a LOAD of it with relocation; the
in-process chain fan-out over two device handles with small chunks."""
import json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_06664_b200 as foundry
from paper_2604_06664_b200 import capi


def step(what):  # progress marker (a sanitizer crash shows where it happened)
    print("step:", what, flush=True)


# `--prepare DIR` writes the two archives (outside the sanitizer: SAVE forks
# ptxas / nvlink, which the sanitizer does not survive after a warm run);
# `DIR` alone runs the case on them.
prepare = sys.argv[1:2] == ["--prepare"]
# `--no-load` skips the LOAD steps (VMM reservations, which initcheck cannot
# follow) and runs fdy_prepare_archive on both layouts instead
no_load = "--no-load" in sys.argv
t = sys.argv[-1] if len(sys.argv) > 1 else tempfile.mkdtemp()
spec = foundry.preset("moe-spmd"); spec.batch_max = 24; spec.thresholds = [5, 9, 17]
if prepare or len(sys.argv) == 1:
    step("save")
    foundry.save(spec, t + "/a")
    foundry.save(spec, t + "/plain", b200_artifacts=False)
    if prepare:
        sys.exit(0)
blob = open(t + "/a/templates.fdt", "rb").read()
base = json.load(open(t + "/a/manifest"))["allocator"]["base"]
api = capi.CApi(); dev = api.device_open(0)
step("materialize")
store = api.store_upload(dev, blob)
m, _ = api.materialize(dev, store, 1, 4, 0)
api.materialize(dev, store, 1, 4, base + 0x10000, m)
step("crc")
api.crc64(dev, blob, [(0, len(blob)), (0, 7), (16, 65536 * 3 + 5)])
api.lib.fdy_members_free(m); api.lib.fdy_store_free(store)
if no_load:
    step("prepare_archive")
    hdr = capi.store_header(blob)
    host = api.host_alloc(dev, hdr["members_image_bytes"])
    for arch in ("/a", "/plain"):
        api.prepare_archive(dev, t + arch, 1, 4, base + 0x10000, 4, host, hdr["members_image_bytes"])
    step("gpu pack")
    gpu, _ = foundry._foundry._pack_store_bytes(t + "/plain", True)
    assert gpu == foundry._foundry._pack_store_bytes(t + "/plain", False)[0]
api.lib.fdy_device_close(dev)
if not no_load:
    step("load device_updates")
    h = foundry.load(t + "/a", rank=1, world=4, device_updates=True)
    for b in h.batches()[:6]:
        h.serve(b); h.replay(b)
    h.close()
    # GPU packer (pack.cu) + a LOAD that packs on the GPU and relocates
    step("gpu pack")
    gpu, _ = foundry._foundry._pack_store_bytes(t + "/plain", True)
    cpu, _ = foundry._foundry._pack_store_bytes(t + "/plain", False)
    assert gpu == cpu
    step("load plain")
    keep = foundry.load(t + "/plain", rank=0, world=4)
    h = foundry.load(t + "/plain", rank=2, world=4, relocate=True)
    for b in h.batches()[:4]:
        h.replay(b)
    h.close(); keep.close()
# chain fan-out (fanout.cu): publish / wait kernels between two streams
step("chain")
dev = api.device_open(0)
devs = [api.device_open(0), api.device_open(0)]
src = api.store_upload(dev, blob)
outs = api.store_fanout_chain(src, devs, 4096 + 16)
for st in outs: api.lib.fdy_store_free(st)
api.lib.fdy_store_free(src)
for d in devs + [dev]: api.lib.fdy_device_close(d)
print("sanitize case ok")
