"""e2e (host arrays in/out) timing of the public spmv() on C2 for several
streamed-path piece layouts, and the Python share of one call."""
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
dm = DeviceMatrix.of(da)
B = 187760644


def timeit(fn, reps=30):
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


layouts = {"eq1": dict(pieces=1), "eq4": dict(pieces=4), "eq8": dict(pieces=8),
           "s16_3": dict(cuts=[1 / 16, 1 / 2, 15 / 16]),
           "s32_5": dict(cuts=[1 / 32, 1 / 4, 1 / 2, 3 / 4, 31 / 32]),
           "s16_4": dict(cuts=[1 / 16, 1 / 3, 2 / 3, 15 / 16]),
           "g8": dict(cuts=[1 / 32, 3 / 32, 1 / 4, 1 / 2, 3 / 4, 29 / 32, 31 / 32])}
for name, kw in layouts.items():
    dm._streamed = hostpath.StreamedHost(dm, **kw)
    el = timeit(lambda: dg.spmv(da, xp.numpy(), yp.numpy()))
    sh = dm._streamed
    xa, ya = xp.numpy(), yp.numpy()
    eld = timeit(lambda: sh.run(xa, ya, 1.0, 0.0, "exact", 0))
    ok = np.array_equal(yp.numpy(), dg.spmv(dm, xp.cuda(), None).cpu().numpy())
    print(f"{name}: spmv() {el*1e3:.3f} ms ({B/el/1e9:.1f} GB/s), run() {eld*1e3:.3f} ms, "
          f"python {1e6*(el-eld):.0f} us, bit-equal {ok}")
