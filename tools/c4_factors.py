"""C4's gap to the stencil class, factor by factor: the 2048^2 5-point
Laplacian in natural order, after scramble -> RCM, and with the Pareto skew
rows on top (= C4); default selection and sliced_pipe, DA and CSR, warm / cold."""
import json
import sys

sys.path.insert(0, ".")
import torch

import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.model import StorageWidths, spmv_traffic
from paper_2307_06305_b200.reorder import permute_symmetric, rcm
from paper_2307_06305_b200.workloads import (add_skew_rows, laplacian_2d, scrambled,
                                             uniform_x)

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["sliced_pipe", "sliced"]
lap = laplacian_2d(nx)
mixed, _ = scrambled(lap, seed=4)
ordered = permute_symmetric(mixed, rcm(mixed))
w = dg.bandwidth(ordered)
skew = add_skew_rows(ordered, frac=0.01, alpha=1.5, x_m=1.0, cap=4096, band=w, seed=5)
x = torch.from_numpy(uniform_x(lap.ncols, 1)).cuda()
for name, a in (("natural", lap), ("rcm", ordered), ("rcm+skew", skew)):
    for kind in ("da", "csr"):
        dm = DeviceMatrix.from_host(dg.to_dacsr(a, 16) if kind == "da" else a)
        tr = spmv_traffic(dm.nrows, dm.ncols, dm.nnz,
                          StorageWidths(dm.oindex_width // 8, dm.iindex_width // 8,
                                        dm.scalar_width // 8)).total_bytes
        y = torch.empty(dm.nrows, dtype=torch.float64, device="cuda")
        for v in variants:
            fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, v, 0)
            warm = time_kernel(fn, epochs=5, warmup_iters=3, min_epoch_iters=3,
                               min_epoch_time=0.05, graph=50)
            cold = time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=8,
                               min_epoch_time=0.0, cold=True)
            print(json.dumps({"matrix": name, "kind": kind, "variant": v,
                              "slices": dm.slices_info() and {k: dm.slices_info()[k] for k in ("max_len", "n_medium", "n_long")},
                              "warm_us": round(warm * 1e6, 2), "cold_us": round(cold * 1e6, 2),
                              "cold_gbs": round(tr / cold / 1e9)}), flush=True)
        del dm
