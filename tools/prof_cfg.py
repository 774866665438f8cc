"""ncu driver: a few SpMVs of one config with one or more kernels.

    python tools/prof_cfg.py c4 sliced,wstream [--reps 2] [--kinds da]

Each launch is preceded by an L2 flush (cold) unless --warm.
"""
import argparse
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import flush_l2
from paper_2307_06305_b200.spmv import kernel_for, resolve_variant
from paper_2307_06305_b200.workloads import laplacian_2d, laplacian_3d, uniform_x

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("variants")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--kinds", default="da")
ap.add_argument("--warm", action="store_true")
ap.add_argument("--max-len", type=int, default=None)
args = ap.parse_args()
dev = torch.device("cuda")
c = args.config
if c == "c4":
    from paper_2307_06305_b200.workloads import skewed_rcm_laplacian
    a, _ = skewed_rcm_laplacian(2048)
    csr, xh = a, uniform_x(a.ncols, 1)
elif c == "c3":
    from paper_2307_06305_b200.gen import banded_device, normal_vector
    mats = banded_device("c3", dev)
    x = normal_vector(mats["da"].ncols, 17, dev)
elif c == "c5slab":  # one 8-GPU rank's share of C5: rows [0, 2^25) (rank 0's slab)
    from paper_2307_06305_b200.gen import banded_device, normal_vector
    mats = banded_device("c5", dev, kinds=tuple(args.kinds.split(",")), r0=0, r1=1 << 25)
    x = normal_vector(1 << 28, 21, dev)
else:
    dt = np.float32 if c == "c2f32" else np.float64
    csr = laplacian_2d(1024, dt) if c == "c1" else laplacian_3d(128, dt)
    xh = uniform_x(csr.ncols, 1).astype(dt)
if c not in ("c3", "c5slab"):
    mats = {"csr": DeviceMatrix.from_host(csr), "da": DeviceMatrix.from_host(dg.to_dacsr(csr, 16))}
    x = torch.from_numpy(xh).to(dev)
    if c == "c2bf16":
        mats = {k: v.astype(torch.bfloat16) for k, v in mats.items()}
        x = x.to(torch.bfloat16)
for kind in args.kinds.split(","):
    dm = mats[kind]
    if args.max_len:
        dm.build_slices(args.max_len)
    y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dev)
    for v in args.variants.split(","):
        k, o = resolve_variant(v)
        k = kernel_for(dm, k, o)
        for _ in range(args.reps):
            if not args.warm:
                flush_l2()
            dm.spmv_into(x, y, 1.0, 0.0, k, o)
torch.cuda.synchronize()
print("ok")
