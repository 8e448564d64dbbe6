"""PCIe ceiling probe behind DESIGN.md section 6: one 4.1 GB pinned H2D copy (the cfg5
input) and H2D + concurrent D2H on two streams.  python tools/h2d_ceiling.py"""
import torch, time
n = 4096800000 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device='cuda')
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
    print('H2D one copy GB/s', 4.0968/ (e0.elapsed_time(e1)/1e3))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
e0.record()
with torch.cuda.stream(s1): d[:n//2].copy_(h[:n//2], non_blocking=True)
with torch.cuda.stream(s2): d[n//2:].copy_(h[n//2:], non_blocking=True)
torch.cuda.synchronize(); 
t0=time.perf_counter(); 
with torch.cuda.stream(s1): d[:n//2].copy_(h[:n//2], non_blocking=True)
with torch.cuda.stream(s2): d[n//2:].copy_(h[n//2:], non_blocking=True)
torch.cuda.synchronize(); print('H2D two streams GB/s', 4.0968/(time.perf_counter()-t0))
m = 1468436508 // 4
hd = torch.empty(m, dtype=torch.float32).pin_memory()
dd = torch.empty(m, dtype=torch.float32, device='cuda')
e0.record(); hd.copy_(dd, non_blocking=True); e1.record(); torch.cuda.synchronize()
print('D2H GB/s', 1.4684/(e0.elapsed_time(e1)/1e3))
# bidirectional
t0=time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): hd.copy_(dd, non_blocking=True)
torch.cuda.synchronize(); print('bidir total s', time.perf_counter()-t0)
