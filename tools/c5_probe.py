"""C5 (2^28 rows, Poisson(8) in [1,32], +-32767 band): sliced layout shape and
per-kernel SpMV times (one SpMV, warm graph of 3)."""
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.gen import banded_arrays, normal_vector
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.workloads import BANDED_CONFIGS

dev = torch.device("cuda")
n, b, lam, kmax, seed = BANDED_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
arr = banded_arrays(n, b, lam, kmax, seed, dev, kinds=("da",))
dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"])
x = normal_vector(n, 21, dev)
y = torch.empty(n, dtype=torch.float64, device=dev)
for ml in (None, 8, 12, 16):
    dm.build_slices(ml)
    info = dm.slices_info()
    t = time_kernel(lambda: dm.spmv_into(x, y, 1.0, 0.0, "sliced", 0), epochs=2, warmup_iters=1,
                    min_epoch_iters=1, min_epoch_time=0.0, graph=3)
    print(json.dumps({"max_len": info["max_len"], "medium": info["n_medium"], "long": info["n_long"],
                      "padding": round(info["padding"], 3), "sliced_ms": round(t * 1e3, 3)}), flush=True)
for k in ("rowblock", "wstream", "scalar"):
    t = time_kernel(lambda: dm.spmv_into(x, y, 1.0, 0.0, k, 0), epochs=2, warmup_iters=1,
                    min_epoch_iters=1, min_epoch_time=0.0, graph=3)
    print(json.dumps({"kernel": k, "ms": round(t * 1e3, 3)}), flush=True)
