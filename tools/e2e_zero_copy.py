"""e2e (host arrays in/out) of the public spmv() on C2: y stored straight
into pinned host memory by the kernels (zero-copy) vs y through a device
buffer + D2H copies (pageable y), for several piece counts and kernels."""
import sys
import time

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
xp = torch.empty(len(x), dtype=torch.float64, pin_memory=True)
xp.numpy()[:] = x
yp = torch.empty(csr.nrows, dtype=torch.float64, pin_memory=True)
ypage = np.empty(csr.nrows)
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


for kernel in ("sliced", "wstream"):
    dm.tuned_kernel = kernel
    for pieces in (1, 2, 4, 8, 16, 32):
        dm._streamed = hostpath.StreamedHost(dm, pieces=pieces)
        for yname, yarr in (("pinned", yp.numpy()), ("pageable", ypage)):
            yarr[:] = 0
            el = timeit(lambda: dg.spmv(da, xp.numpy(), yarr))
            ok = np.array_equal(yarr.view(np.uint64), ref.view(np.uint64))
            print(f"{kernel} pieces={pieces} y={yname}: {el*1e3:.3f} ms "
                  f"({B/el/1e9:.1f} GB/s) bit-equal {ok}", flush=True)
