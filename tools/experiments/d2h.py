# D2H ceiling for the e2e output size (147 MB) into pinned memory: one copy vs split across streams
import torch, time
n = 147161088
d = torch.empty(n, dtype=torch.uint8, device="cuda").fill_(1)
h = torch.empty(n, dtype=torch.uint8).pin_memory()
ss = [torch.cuda.Stream() for _ in range(4)]
def run(k, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter()
        step = (n + k - 1) // k
        for i in range(k):
            with torch.cuda.stream(ss[i]):
                h[i*step:(i+1)*step].copy_(d[i*step:(i+1)*step], non_blocking=True)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    print(f"D2H 147 MB split {k}: {best*1e3:.3f} ms  {n/best/1e9:.1f} GB/s")
for k in (1, 2, 4, 1):
    run(k)
hp = torch.empty(n, dtype=torch.uint8)  # pageable
torch.cuda.synchronize(); t = time.perf_counter(); hp.copy_(d); torch.cuda.synchronize(); print("pageable D2H", (time.perf_counter()-t)*1e3, "ms")
