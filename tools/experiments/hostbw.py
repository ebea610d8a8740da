import torch, time
torch.set_num_threads(16)
a=torch.ones(1<<30,dtype=torch.uint8); b=torch.empty_like(a)
for i in range(3):
    t=time.perf_counter(); b.copy_(a); dt=time.perf_counter()-t; print("host copy 1GiB", dt*1e3, "ms", 2*(1<<30)/dt/1e9, "GB/s (r+w)")
for i in range(3):
    t=time.perf_counter(); s=a.sum(dtype=torch.int64); dt=time.perf_counter()-t; print("host read 1GiB", dt*1e3, "ms", (1<<30)/dt/1e9, "GB/s")
p=torch.empty(256<<20,dtype=torch.uint8).pin_memory(); d=torch.empty(256<<20,dtype=torch.uint8,device="cuda"); q=torch.empty(256<<20,dtype=torch.uint8).pin_memory()
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(p,non_blocking=True)
    torch.cuda.synchronize(); t1=time.perf_counter()-t
    t=time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(p,non_blocking=True)
    with torch.cuda.stream(s2): q.copy_(d,non_blocking=True)
    torch.cuda.synchronize(); t2=time.perf_counter()-t
    print("H2D 256MiB alone %.2f ms; H2D+D2H concurrently %.2f ms"%(t1*1e3,t2*1e3))
# H2D while host copies run
import threading
def hostwork():
    for _ in range(3): b.copy_(a)
th=threading.Thread(target=hostwork); th.start()
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(4): d.copy_(p,non_blocking=True)
torch.cuda.synchronize(); dt=time.perf_counter()-t; th.join()
print("H2D 1GiB under host copy load: %.2f ms (%.1f GB/s)"%(dt*1e3,(1<<30)/dt/1e9))
