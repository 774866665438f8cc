"""Experiment: the SpMV kernel reading x from and writing y to pinned host
memory directly (UVA, no copies at all), C2, against the streamed path."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.workloads import laplacian_3d, uniform_x

csr = laplacian_3d(128)
da = dg.to_dacsr(csr, 16)
x = uniform_x(csr.ncols, 1)
xp = torch.empty(len(x), dtype=torch.float64, pin_memory=True)
xp.numpy()[:] = x
yp = torch.empty(csr.nrows, dtype=torch.float64, pin_memory=True)
dm = DeviceMatrix.of(da)
dm.build_slices()
B = 187760644
ref = dg.spmv(dm, xp.cuda(), None).cpu().numpy()


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        best = min(best, (time.perf_counter() - t0) / reps)
    return best


for kernel in ("sliced", "wstream", "scalar"):
    def direct():
        dm.spmv_into(xp, yp, 1.0, 0.0, kernel, 0)
        torch.cuda.current_stream().synchronize()
    yp.numpy()[:] = 0
    el = timeit(direct)
    ok = np.array_equal(yp.numpy().view(np.uint64), ref.view(np.uint64))
    print(f"direct {kernel}: {el*1e3:.3f} ms ({B/el/1e9:.1f} GB/s) bit-equal {ok}", flush=True)
    dm.tuned_kernel = kernel
    el = timeit(lambda: dg.spmv(da, xp.numpy(), yp.numpy()))
    print(f"streamed {kernel}: {el*1e3:.3f} ms ({B/el/1e9:.1f} GB/s)", flush=True)
