import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_1507_08101_b200 import sellkit
sk = sellkit.load()
n, w = int(sys.argv[1]), 8
N = n**3
A = sk.crs_stencil(7, n).build(32, 256)
xh = torch.empty((N, w), dtype=torch.float64, pin_memory=True)
yh = torch.empty((N, w), dtype=torch.float64, pin_memory=True)
xh.uniform_()
xv = sk.view_plain(xh.data_ptr(), N*w, N, w, w, keep=xh)
yv = sk.view_plain(yh.data_ptr(), N*w, N, w, w, keep=yh)
for i in range(3):
    t0 = time.perf_counter(); sk.spmv(yv, A, xv); t1 = time.perf_counter()
    print(f"streamed host spmv n={n}: {(t1-t0)*1e3:.1f} ms  -> {2*(7*N-6*n*n)*w/(t1-t0)/1e9:.1f} GF/s", flush=True)
# raw copy bandwidth
xd = torch.empty((N, w), dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); xd.copy_(xh, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"H2D {N*w*8/(t1-t0)/1e9:.1f} GB/s"); t0 = time.perf_counter(); yh.copy_(xd, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"D2H {N*w*8/(t1-t0)/1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
yd = torch.empty_like(xd)
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): xd.copy_(xh, non_blocking=True)
with torch.cuda.stream(s2): yh.copy_(yd, non_blocking=True)
torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"bidirectional {2*N*w*8/(t1-t0)/1e9:.1f} GB/s total")
