"""WSTREAM 32- vs 64-row chunks (planner window for each) on C1, C2, C4."""
import sys
sys.path.insert(0, ".")
import json
import numpy as np
import torch
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.model import StorageWidths, spmv_traffic
from paper_2307_06305_b200.workloads import laplacian_2d, laplacian_3d, skewed_rcm_laplacian, uniform_x

dev = torch.device("cuda")
for c in sys.argv[1].split(","):
    if c == "c4":
        csr = skewed_rcm_laplacian(2048)[0]
    else:
        csr = laplacian_2d(1024) if c == "c1" else laplacian_3d(128)
    for kind, a in (("da", dg.to_dacsr(csr, 16)), ("csr", csr)):
        dm = DeviceMatrix.from_host(a)
        x = torch.from_numpy(uniform_x(csr.ncols, 1)).to(dev)
        tr = spmv_traffic(dm.nrows, dm.ncols, dm.nnz, StorageWidths(4, dm.iindex_width // 8, 8)).total_bytes
        y = torch.empty(dm.nrows, dtype=torch.float64, device=dev)
        ref = None
        for rows in (32, 64):
            vcap = dm.chunk_window(rows)
            dm.set_chunk_window(vcap, rows)
            fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, "wstream", 0)
            fn()
            if ref is None:
                ref = y.clone()
            ok = bool(torch.equal(ref, y))
            warm = time_kernel(fn, epochs=5, warmup_iters=3, min_epoch_iters=3, min_epoch_time=0.05, graph=20)
            cold = time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=5, min_epoch_time=0.0, cold=True)
            p = dm.chunk_plan(vcap, rows)
            print(json.dumps({"config": c, "kind": kind, "rows": rows, "vcap": vcap, "complex": p.n_complex,
                              "bit_equal": ok, "warm_us": round(warm * 1e6, 2), "warm_gbs": round(tr / warm / 1e9),
                              "cold_us": round(cold * 1e6, 2), "cold_gbs": round(tr / cold / 1e9)}), flush=True)
