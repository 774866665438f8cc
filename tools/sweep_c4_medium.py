"""C4: sliced-kernel time vs the medium/long split (max_len, medium_len)."""
import json
import sys

sys.path.insert(0, ".")
import torch

import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.workloads import skewed_rcm_laplacian, uniform_x

a, _ = skewed_rcm_laplacian(2048)
dm = DeviceMatrix.from_host(dg.to_dacsr(a, 16))
x = torch.from_numpy(uniform_x(a.ncols, 1)).cuda()
y = torch.empty(a.nrows, dtype=torch.float64, device="cuda")
for ml, med in ((6, 8), (6, 16), (6, 24), (6, 32), (6, 64), (6, 128), (5, 32), (8, 16), (8, 32), (8, 64), (12, 32), (16, 32)):
    dm.build_slices(ml, med)
    info = dm.slices_info()
    fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, "sliced_pipe", 0)
    warm = time_kernel(fn, epochs=3, warmup_iters=3, min_epoch_iters=5, min_epoch_time=0.02, graph=20)
    print(json.dumps({"max_len": ml, "medium_len": med, "n_medium": info["n_medium"],
                      "n_long": info["n_long"], "warm_us": round(warm * 1e6, 2)}), flush=True)
