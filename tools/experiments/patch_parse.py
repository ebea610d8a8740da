"""Time parse_patch_view on the headline patch.bin, alone and while 16 threads
stream graphs.bin from the page cache (the e2e_plain contention)."""
import os, sys, time, threading
sys.path.insert(0, os.getcwd())
import paper_2604_06664_b200 as foundry
root = "/tmp/foundry_bench_qwen3-235b-a22b/plain"
if not os.path.exists(root + "/patch.bin"):
    w = foundry.workload_from_text(open(foundry.workload_path("qwen3-235b-a22b")).read())
    foundry.save(w, root, b200_artifacts=False)
raw = open(root + "/patch.bin", "rb").read()
for i in range(5):
    t0 = time.perf_counter(); foundry._foundry._parse_patch_view(raw); print("alone %.3f ms" % ((time.perf_counter() - t0) * 1e3))
stop = False
def reader():
    fd = os.open(root + "/graphs.bin", os.O_RDONLY)
    while not stop:
        os.pread(fd, 2 << 20, 0)
    os.close(fd)
ts = [threading.Thread(target=reader) for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8)]
for t in ts: t.start()
time.sleep(0.2)
for i in range(5):
    t0 = time.perf_counter(); foundry._foundry._parse_patch_view(raw); print("contended %.3f ms" % ((time.perf_counter() - t0) * 1e3))
stop = True
for t in ts: t.join()
