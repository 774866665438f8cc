"""e2e (pinned host x / y) timing of the public spmv() on C3 for several
streamed-path piece counts (hostpath.StreamedHost)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200 import hostpath
from paper_2307_06305_b200.gen import banded_device, normal_vector

dm = banded_device("c3", "cuda", kinds=("da",))["da"]
x = normal_vector(dm.ncols, 17, "cuda")
xp = torch.empty(dm.ncols, dtype=torch.float64, pin_memory=True)
xp.copy_(x)
yp = torch.empty(dm.nrows, dtype=torch.float64, pin_memory=True)
B = 3017661244
ref = dg.spmv(dm, x, None).cpu().numpy()


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        best = min(best, (time.perf_counter() - t0) / reps)
    return best


for pieces in [int(a) for a in sys.argv[1:]] or [1, 4, 8, 16, 32, 64]:
    for through in (0, 1):
        dm._streamed = hostpath.StreamedHost(dm, pieces=pieces, y_through_device=through)
        el = timeit(lambda: dg.spmv(dm, xp.numpy(), yp.numpy()))
        ok = np.array_equal(yp.numpy(), ref)
        print(f"pieces {pieces} y_through_device {through}: {el*1e3:.3f} ms per spmv "
              f"({B/el/1e9:.1f} GB/s), bit-equal {ok}", flush=True)
