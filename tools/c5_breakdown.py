"""C5 power-iteration time breakdown on one GPU (GPU box):
full-range SpMV vs interior + two boundary strips (the distributed launch
pattern) vs the deterministic norm (sumsq chunks + ordered fold + host read).

    python tools/c5_breakdown.py
"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2307_06305_b200 import distributed as D
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.gen import banded_arrays, normal_vector
from paper_2307_06305_b200.power import chunk_partials, fold_ordered, partials_from_groups
from paper_2307_06305_b200.workloads import BANDED_CONFIGS

dev = torch.device("cuda")
n, b, lam, kmax, seed = BANDED_CONFIGS["c5"]
arr = banded_arrays(n, b, lam, kmax, seed, dev, kinds=("da",))
dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"])
x = normal_vector(n, 21, dev)
y = torch.empty(n, dtype=torch.float64, device=dev)
dm.spmv_into(x, y, 1.0, 0.0, "tiled")
torch.cuda.synchronize()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"nnz": dm.nnz}
out["spmv_full_ms"] = timed(lambda: dm.spmv_into(x, y, 1.0, 0.0, "tiled"))
cut0, cut1 = b, n - b
out["spmv_interior_ms"] = timed(lambda: dm.spmv_into(x, y, 1.0, 0.0, "tiled", row_start=cut0,
                                                     row_end=cut1))
out["spmv_strip_ms"] = timed(lambda: dm.spmv_into(x, y, 1.0, 0.0, "tiled", row_start=0,
                                                  row_end=cut0))
alpha = torch.ones(1, dtype=torch.float64, device=dev)
gs = torch.empty((n + 511) // 512, dtype=torch.float64, device=dev)
out["spmv_full_fused_sumsq_ms"] = timed(lambda: dm.spmv_into(x, y, alpha, 0.0, "tiled",
                                                              group_sumsq=gs))
out["partials_from_groups_ms"] = timed(lambda: partials_from_groups(gs, n, 1 << 16))
out["sumsq_chunks_ms"] = timed(lambda: chunk_partials(y, 1 << 16))
p = chunk_partials(y, 1 << 16)
out["fold_ordered_ms"] = timed(lambda: fold_ordered(p))
t0 = time.perf_counter()
for _ in range(20):
    float(fold_ordered(chunk_partials(y, 1 << 16)).item())
out["norm_with_host_read_ms"] = (time.perf_counter() - t0) / 20 * 1e3
print(json.dumps(out), flush=True)
