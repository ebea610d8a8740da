import os, time, torch, glob, threading
from concurrent.futures import ThreadPoolExecutor
A="/tmp/foundry_bench_qwen3-235b-a22b/b200"
files=[f for f in glob.glob(A+"/**",recursive=True) if os.path.isfile(f)]
tot=sum(os.path.getsize(f) for f in files); print("files",len(files),"bytes",tot, "cpus", os.cpu_count())
pin=torch.empty(tot+len(files)*4096,dtype=torch.uint8).pin_memory()
dev=torch.empty_like(pin,device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); dev.copy_(pin,non_blocking=True); torch.cuda.synchronize(); print("H2D all", (time.perf_counter()-t)*1e3, "ms")
    t=time.perf_counter(); pin[:147161088].copy_(dev[:147161088],non_blocking=True); torch.cuda.synchronize(); print("D2H 147MB", (time.perf_counter()-t)*1e3, "ms")
mv=memoryview(pin.numpy())
pieces=[]; off=0
for f in files:
    n=os.path.getsize(f)
    for o in range(0,n,8<<20): pieces.append((f,o,min(8<<20,n-o),off+o))
    off+=(n+4095)//4096*4096
def rd(p):
    f,o,n,d=p
    fd=os.open(f,os.O_RDONLY); os.preadv(fd,[mv[d:d+n]],o); os.close(fd)
for lanes in (4,8,16,32):
    with ThreadPoolExecutor(lanes) as ex:
        t=time.perf_counter(); list(ex.map(rd,pieces)); print("read lanes",lanes,(time.perf_counter()-t)*1e3,"ms")
