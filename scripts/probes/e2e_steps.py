import time, sys, os
sys.path.insert(0, os.getcwd())
import torch
from gen import hgen
from paper_2008_12441_b200 import hmat as hm
cfg = hgen.CONFIGS["c4"]
h = hm.hmat_create_uninit(cfg.L, cfg.d, cfg.b, cfg.r)
n = cfg.N
xh = [torch.rand(n, dtype=torch.float64).pin_memory() for _ in range(2)]
yh = torch.empty(n, dtype=torch.float64).pin_memory()
xd = torch.rand(n, dtype=torch.float64, device="cuda"); yd = torch.empty_like(xd)
for _ in range(5): hm.hmat_matvec(h, xd, yd)
torch.cuda.synchronize()
t0=time.perf_counter()
for i in range(40): hm.hmat_matvec(h, xd, yd)
torch.cuda.synchronize(); print("device", (time.perf_counter()-t0)/40*1e3)
hm.hmat_set_host_async(h, True)
hm.hmat_matvec(h, xh[0], yh); hm.hmat_synchronize(h)
for K in (8, 20, 64, 128):
    t0=time.perf_counter()
    for i in range(K): hm.hmat_matvec(h, xh[i%2], yh)
    hm.hmat_synchronize(h)
    print("async", K, (time.perf_counter()-t0)/K*1e3)
