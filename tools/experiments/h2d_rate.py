import torch, time
n = 188 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    print("H2D 188MB one copy %.2f ms" % ((time.perf_counter() - t) * 1e3))
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    for k in range(94):
        d[k * (2 << 20):(k + 1) * (2 << 20)].copy_(h[k * (2 << 20):(k + 1) * (2 << 20)], non_blocking=True)
    torch.cuda.synchronize()
    print("H2D 94 x 2MB %.2f ms" % ((time.perf_counter() - t) * 1e3))
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    print("D2H 188MB %.2f ms" % ((time.perf_counter() - t) * 1e3))
