"""Host overhead of one public spmv() call (small matrix, host arrays), with
a cProfile breakdown."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.workloads import laplacian_3d, uniform_x
small = dg.to_dacsr(laplacian_3d(8), 16)
xs = uniform_x(small.ncols, 1)
ys = np.empty(small.nrows)
for _ in range(20):
    dg.spmv(small, xs, ys)
t0 = time.perf_counter()
for _ in range(500):
    dg.spmv(small, xs, ys)
print(f"host arrays: {(time.perf_counter()-t0)/500*1e6:.1f} us/call")
dm = dg.DeviceMatrix.of(small)
xd = torch.from_numpy(xs).cuda(); yd = torch.empty(small.nrows, dtype=torch.float64, device="cuda")
for _ in range(20):
    dg.spmv(dm, xd, yd)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500):
    dg.spmv(dm, xd, yd)
torch.cuda.synchronize()
print(f"device tensors: {(time.perf_counter()-t0)/500*1e6:.1f} us/call")
t0 = time.perf_counter()
for _ in range(500):
    dm.spmv_into(xd, yd, 1.0, 0.0, "wstream", 0)
torch.cuda.synchronize()
print(f"spmv_into: {(time.perf_counter()-t0)/500*1e6:.1f} us/call")
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    dg.spmv(small, xs, ys)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
