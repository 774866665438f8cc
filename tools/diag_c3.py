"""C3 (random band): per-kernel cold / warm time of every exact kernel, with
progress timestamps (diagnosed the harness over-enqueue that made warm
timings of millisecond SpMVs take minutes)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2307_06305_b200.gen import banded_device, normal_vector
from paper_2307_06305_b200.harness import time_kernel
t0 = time.time()
def log(*a):
    print(f"[{time.time()-t0:7.1f}s]", *a, flush=True)
dev = torch.device("cuda")
mats = banded_device("c3", dev)
x = normal_vector(mats["da"].ncols, 17, dev)
log("built")
for kind in ("da", "csr"):
    dm = mats[kind]
    y = torch.empty(dm.nrows, dtype=torch.float64, device=dev)
    for v in sys.argv[1].split(","):
        log(kind, v, "first launch")
        dm.spmv_into(x, y, 1.0, 0.0, v, 0)
        torch.cuda.synchronize()
        log(kind, v, "ok; cold timing")
        t = time_kernel(lambda: dm.spmv_into(x, y, 1.0, 0.0, v, 0), epochs=2, warmup_iters=1, min_epoch_iters=3, min_epoch_time=0.0, cold=True)
        log(kind, v, f"cold {t*1e3:.3f} ms; warm graph")
        t = time_kernel(lambda: dm.spmv_into(x, y, 1.0, 0.0, v, 0), epochs=2, warmup_iters=1, min_epoch_iters=2, min_epoch_time=0.01, graph=10)
        log(kind, v, f"warm {t*1e3:.3f} ms")
