import numpy as np, time, ctypes, os, torch
from concurrent.futures import ThreadPoolExecutor
print("cpus", len(os.sched_getaffinity(0)), os.cpu_count())
n=51_381_960
src=np.frombuffer(np.random.bytes(n),np.uint8)
pinned=torch.empty(n, dtype=torch.uint8, pin_memory=True); pd=pinned.numpy(); pd[:]=0
dst=np.empty(n,np.uint8); dst[:]=0
for label, d in (("pinned", pd), ("pageable", dst)):
    sa=src.ctypes.data; da=d.ctypes.data
    for C in (2<<20, 8<<20):
        bounds=list(range(0,n,C))+[n]
        for nt in (1,2,4,8,16):
            pool=ThreadPoolExecutor(nt)
            def f1(c): ctypes.memmove(da+bounds[c], sa+bounds[c], bounds[c+1]-bounds[c])
            def f2(c): d[bounds[c]:bounds[c+1]]=src[bounds[c]:bounds[c+1]]
            out=[]
            for f in (f1,f2):
                ts=[]
                for r in range(9):
                    t=time.perf_counter(); list(pool.map(f, range(len(bounds)-1))); ts.append(time.perf_counter()-t)
                out.append(np.median(ts)*1e3)
            print(label, C>>20, "MB", nt, "memmove %.2f numpy %.2f ms"%tuple(out))
