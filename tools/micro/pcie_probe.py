import torch
n=1<<25  # 32M doubles = 256 MiB
h=torch.empty(n,dtype=torch.float64).pin_memory(); d=torch.empty(n,dtype=torch.float64,device='cuda')
h2=torch.empty(n//2,dtype=torch.float64).pin_memory()
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/reps
ms=t(lambda: d.copy_(h, non_blocking=True)); print("H2D 256MiB single", ms, "ms", n*8/ms/1e6, "GB/s")
ms=t(lambda: h.copy_(d, non_blocking=True)); print("D2H 256MiB single", ms, "ms", n*8/ms/1e6, "GB/s")
def two():
    cur=torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d[:n//2].copy_(h[:n//2], non_blocking=True)
    with torch.cuda.stream(s2): d[n//2:].copy_(h[n//2:], non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
ms=t(two); print("H2D 2 streams", ms, "ms", n*8/ms/1e6, "GB/s")
def bidir():
    cur=torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d[:n//2].copy_(h[:n//2], non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d[n//2:], non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
ms=t(bidir); print("H2D 128MiB || D2H 128MiB", ms, "ms")
