import json, sys
sys.path.insert(0, ".")
import torch
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.reorder import permute_symmetric, rcm
from paper_2307_06305_b200.workloads import add_skew_rows, laplacian_2d, scrambled, uniform_x
lap = laplacian_2d(2048)
mixed, _ = scrambled(lap, seed=4)
ordered = permute_symmetric(mixed, rcm(mixed))
w = dg.bandwidth(ordered)
x = torch.from_numpy(uniform_x(lap.ncols, 1)).cuda()
for cap in (1, 3, 27, 4096):
    a = add_skew_rows(ordered, frac=0.01, alpha=1.5, x_m=1.0, cap=cap, band=w, seed=5)
    dm = DeviceMatrix.from_host(dg.to_dacsr(a, 16))
    y = torch.empty(dm.nrows, dtype=torch.float64, device="cuda")
    fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, "sliced_pipe", 0)
    warm = time_kernel(fn, epochs=5, warmup_iters=3, min_epoch_iters=3, min_epoch_time=0.05, graph=50)
    info = dm.slices_info()
    print(json.dumps({"cap": cap, "nnz": dm.nnz, "max_len": info["max_len"], "n_medium": info["n_medium"], "n_long": info["n_long"], "slots": info["slots"], "warm_us": round(warm * 1e6, 2)}), flush=True)
