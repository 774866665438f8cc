"""e2e (host arrays in/out) timing of the public spmv() on C2 for several
streamed-path piece counts; also checks is_pinned propagation."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200 import hostpath
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.workloads import laplacian_3d, uniform_x

csr = laplacian_3d(128)
da = dg.to_dacsr(csr, 16)
x = uniform_x(csr.ncols, 1)
xp = torch.empty(len(x), dtype=torch.float64, pin_memory=True); xp.numpy()[:] = x
yp = torch.empty(csr.nrows, dtype=torch.float64, pin_memory=True)
print("from_numpy pinned:", torch.from_numpy(xp.numpy()).is_pinned())
dm = DeviceMatrix.of(da)
for pieces in (1, 2, 4, 8, 16):
    dm._streamed = hostpath.StreamedHost(dm, pieces)
    for _ in range(3):
        dg.spmv(da, xp.numpy(), yp.numpy())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        dg.spmv(da, xp.numpy(), yp.numpy())
    el = (time.perf_counter() - t0) / 20
    print(f"pieces={pieces}: {el*1e3:.3f} ms per call, {187760644/el/1e9:.1f} GB/s")
# host-side overhead of one call with a tiny matrix
small = dg.to_dacsr(laplacian_3d(8), 16)
xs = uniform_x(small.ncols, 1)
for _ in range(10):
    dg.spmv(small, xs)
t0 = time.perf_counter()
for _ in range(200):
    dg.spmv(small, xs)
print(f"small call overhead {(time.perf_counter()-t0)/200*1e6:.1f} us")
