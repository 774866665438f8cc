"""Sweep the sliced kernel's knobs: resident CTAs per SM and the slice
max_len (spill threshold), on C2 / C2-f32 / C4 (DA)."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.model import StorageWidths, spmv_traffic
from paper_2307_06305_b200.workloads import laplacian_3d, skewed_rcm_laplacian, uniform_x

dev = torch.device("cuda")
CAPS = tuple(int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "0").split(","))
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["sliced"]
for c in (sys.argv[1] if len(sys.argv) > 1 else "c2,c2f32,c4").split(","):
    if c == "c4":
        a, _ = skewed_rcm_laplacian(2048)
        xh = uniform_x(a.ncols, 1)
        lens = (None, 5, 6, 8)
    else:
        dt = np.float32 if c == "c2f32" else np.float64
        a = laplacian_3d(128, dt)
        xh = uniform_x(a.ncols, 1).astype(dt)
        lens = (None,)
    dm = DeviceMatrix.from_host(dg.to_dacsr(a, 16))
    x = torch.from_numpy(xh).to(dev)
    tr = spmv_traffic(dm.nrows, dm.ncols, dm.nnz, StorageWidths(4, 2, dm.scalar_width // 8)).total_bytes
    y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dev)
    for ml in lens:
        dm.build_slices(ml)
        info = dm.slices_info()
        for cap in CAPS:
            dm.set_ctas_per_sm(cap)
            for v in variants:
                fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, v, 0)
                warm = time_kernel(fn, epochs=5, warmup_iters=3, min_epoch_iters=3, min_epoch_time=0.05, graph=50)
                cold = time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=8, min_epoch_time=0.0, cold=True)
                print(json.dumps({"config": c, "variant": v, "max_len": info["max_len"],
                                  "medium": info["n_medium"], "long": info["n_long"], "pad": round(info["padding"], 4),
                                  "ctas_per_sm": cap, "warm_us": round(warm * 1e6, 2),
                                  "warm_gbs": round(tr / warm / 1e9), "cold_us": round(cold * 1e6, 2)}),
                      flush=True)
