"""Sweep WSTREAM's resident CTAs per SM on C2 (f64, f32) and C1/C4/C3."""
import sys
sys.path.insert(0, ".")
import json
import numpy as np
import torch
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.gen import banded_device, normal_vector
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.model import StorageWidths, spmv_traffic
from paper_2307_06305_b200.workloads import laplacian_2d, laplacian_3d, uniform_x

dev = torch.device("cuda")
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2", "c2f32", "c1"]
for c in cfgs:
    if c == "c3":
        dm = banded_device("c3", dev, kinds=("da",))["da"]
        x = normal_vector(dm.ncols, 17, dev)
    else:
        dt = np.float32 if c == "c2f32" else np.float64
        csr = laplacian_2d(1024, dt) if c == "c1" else laplacian_3d(128, dt)
        dm = DeviceMatrix.from_host(dg.to_dacsr(csr, 16))
        x = torch.from_numpy(uniform_x(csr.ncols, 1).astype(dt)).to(dev)
    tr = spmv_traffic(dm.nrows, dm.ncols, dm.nnz, StorageWidths(dm.oindex_width // 8, 2, dm.scalar_width // 8)).total_bytes
    y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dev)
    for cap in (1, 2, 3, 4, 0):
        dm.set_ctas_per_sm(cap)
        fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, "wstream", 0)
        warm = time_kernel(fn, epochs=5, warmup_iters=3, min_epoch_iters=3, min_epoch_time=0.05, graph=20)
        cold = time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=5, min_epoch_time=0.0, cold=True)
        print(json.dumps({"config": c, "ctas_per_sm": cap, "warm_us": round(warm * 1e6, 2),
                          "warm_gbs": round(tr / warm / 1e9), "cold_us": round(cold * 1e6, 2),
                          "cold_gbs": round(tr / cold / 1e9)}), flush=True)
