"""Small driver for ncu: a few SpMVs of config C2 (DA and CSR) with one kernel."""
import argparse
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import flush_l2
from paper_2307_06305_b200.spmv import kernel_for, resolve_variant
from paper_2307_06305_b200.workloads import laplacian_3d, uniform_x

ap = argparse.ArgumentParser()
ap.add_argument("--variants", default="naive")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--kinds", default="da,csr")
args = ap.parse_args()
csr = laplacian_3d(128)
mats = {"da": DeviceMatrix.from_host(dg.to_dacsr(csr, 16)), "csr": DeviceMatrix.from_host(csr)}
x = torch.from_numpy(uniform_x(csr.ncols, 1)).cuda()
y = torch.empty(csr.nrows, dtype=torch.float64, device="cuda")
for kind in args.kinds.split(","):
    dm = mats[kind]
    for v in args.variants.split(","):
        k, o = resolve_variant(v)
        k = kernel_for(dm, k, o)
        for _ in range(args.reps):
            flush_l2()
            dm.spmv_into(x, y, 1.0, 0.0, k, o)
torch.cuda.synchronize()
print("ok")
