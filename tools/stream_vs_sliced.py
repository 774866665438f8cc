"""WSTREAM against SLICED_PIPE on stencil matrices of growing size (where is
the crossover?): warm = graph of 10 back-to-back SpMVs, cold = L2 flushed.

    python tools/stream_vs_sliced.py
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.model import StorageWidths, spmv_traffic
from paper_2307_06305_b200.workloads import laplacian_2d, laplacian_3d_box, uniform_x

dev = torch.device("cuda")
CASES = [("3d 128x128x128", lambda: laplacian_3d_box((128, 128, 128))),
         ("3d 256x128x128", lambda: laplacian_3d_box((256, 128, 128))),
         ("3d 512x128x128", lambda: laplacian_3d_box((512, 128, 128))),
         ("3d 1024x128x128", lambda: laplacian_3d_box((1024, 128, 128))),
         ("3d 1024x128x128 f32", lambda: laplacian_3d_box((1024, 128, 128), np.float32)),
         ("2d 2048^2", lambda: laplacian_2d(2048)),
         ("2d 4096^2", lambda: laplacian_2d(4096))]
only = sys.argv[1] if len(sys.argv) > 1 else ""
for name, build in CASES:
    if only not in name:
        continue
    csr = build()
    mats = {"da": DeviceMatrix.from_host(dg.to_dacsr(csr, 16)), "csr": DeviceMatrix.from_host(csr)}
    x = torch.from_numpy(uniform_x(csr.ncols, 1).astype(csr.values.dtype)).to(dev)
    for kind, dm in mats.items():
        tr = spmv_traffic(dm.nrows, dm.ncols, dm.nnz, StorageWidths(
            dm.oindex_width // 8, dm.iindex_width // 8, dm.scalar_width // 8)).total_bytes
        y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dev)
        rec = {"case": name, "kind": kind, "rows": dm.nrows, "MB": round(tr / 1e6)}
        for k in ("sliced_pipe", "sliced", "wstream") * 2:
            fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, k, 0)
            warm = time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=3, min_epoch_time=0.0,
                               graph=10)
            cold = time_kernel(fn, epochs=3, warmup_iters=1, min_epoch_iters=4, min_epoch_time=0.0,
                               cold=True)
            prev = rec.get(k)
            rec[k] = {"warm_us": round(warm * 1e6, 1), "cold_us": round(cold * 1e6, 1),
                      "warm_gbs": round(tr / warm / 1e9), "cold_gbs": round(tr / cold / 1e9)}
            if prev:  # second pass: keep both
                rec[k]["first_pass"] = [prev["warm_us"], prev["cold_us"]]
        print(json.dumps(rec), flush=True)
    del mats
    torch.cuda.empty_cache()
