import sys, json
sys.path.insert(0, ".")
import torch
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.gen import banded_arrays, normal_vector
from paper_2307_06305_b200.workloads import BANDED_CONFIGS
dev = torch.device("cuda")
n, b, lam, kmax, seed = BANDED_CONFIGS["c5"]
arr = banded_arrays(n, b, lam, kmax, seed, dev, kinds=("da",))
dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"])
x = normal_vector(n, 21, dev)
y = torch.empty(n, dtype=torch.float64, device=dev)
alpha = torch.ones(1, dtype=torch.float64, device=dev)
gs = torch.empty((n + 511) // 512, dtype=torch.float64, device=dev)
def timed(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps
fns = {"host_alpha": lambda: dm.spmv_into(x, y, 1.0, 0.0, "tiled"),
       "dev_alpha": lambda: dm.spmv_into(x, y, alpha, 0.0, "tiled"),
       "dev_alpha_fused": lambda: dm.spmv_into(x, y, alpha, 0.0, "tiled", group_sumsq=gs)}
for rnd in range(4):
    print({k: round(timed(f), 3) for k, f in fns.items()}, flush=True)
