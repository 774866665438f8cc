"""Time one kernel variant across configs for each A/B library build.

    python tools/ab_run.py --variant sliced --configs c2,c2f32 base build/ab/x/libdacsr_b200.so ...

Each library runs in its own subprocess (DACSR_LIB_PATH); "base" is the
in-tree build.  Prints one JSON line per (library, config, kind).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.model import StorageWidths, spmv_traffic
from paper_2307_06305_b200.workloads import laplacian_2d, laplacian_3d, uniform_x
tag, variant, configs, kinds = sys.argv[1], sys.argv[2], sys.argv[3].split(","), sys.argv[4].split(",")
dev = torch.device("cuda")
for c in configs:
    if c == "c3":
        from paper_2307_06305_b200.gen import banded_device, normal_vector
        mats = banded_device("c3", dev)
        x = normal_vector(mats["da"].ncols, 17, dev)
    elif c == "c4":
        from paper_2307_06305_b200.workloads import skewed_rcm_laplacian
        a, _ = skewed_rcm_laplacian(2048)
        mats = {"csr": DeviceMatrix.from_host(a), "da": DeviceMatrix.from_host(dg.to_dacsr(a, 16))}
        x = torch.from_numpy(uniform_x(a.ncols, 1)).to(dev)
    else:
        dt = {"c2f32": np.float32, "c2xlf32": np.float32}.get(c, np.float64)
        if c in ("c2xl", "c2xlf32"):  # C2's stencil, int16 offsets, 8x the rows: out of L2
            from paper_2307_06305_b200.workloads import laplacian_3d_box
            csr = laplacian_3d_box((1024, 128, 128), dt)
        else:
            csr = laplacian_2d(1024, dt) if c == "c1" else laplacian_3d(128, dt)
        mats = {"csr": DeviceMatrix.from_host(csr), "da": DeviceMatrix.from_host(dg.to_dacsr(csr, 16))}
        x = torch.from_numpy(uniform_x(csr.ncols, 1).astype(dt)).to(dev)
        if c == "c2bf16":
            mats = {k: v.astype(torch.bfloat16) for k, v in mats.items()}
            x = x.to(torch.bfloat16)
    for kind in kinds:
        dm = mats[kind]
        tr = spmv_traffic(dm.nrows, dm.ncols, dm.nnz, StorageWidths(dm.oindex_width // 8, dm.iindex_width // 8, dm.scalar_width // 8)).total_bytes
        y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dev)
        fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, variant, 0)
        warm = time_kernel(fn, epochs=5, warmup_iters=3, min_epoch_iters=3, min_epoch_time=0.05, graph=50)
        cold = time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=8, min_epoch_time=0.0, cold=True)
        y2 = torch.empty_like(y)
        dm.spmv_into(x, y2, 1.0, 0.0, "scalar", 0)
        fn()
        exact = bool(torch.equal(y.view(torch.int16) if y.element_size() == 2 else y.view(torch.int32 if y.element_size() == 4 else torch.int64),
                                 y2.view(torch.int16) if y.element_size() == 2 else y2.view(torch.int32 if y.element_size() == 4 else torch.int64)))
        print(json.dumps({"lib": tag, "config": c, "kind": kind, "variant": variant, "exact": exact,
                          "warm_us": round(warm * 1e6, 2), "warm_gbs": round(tr / warm / 1e9),
                          "cold_us": round(cold * 1e6, 2), "cold_gbs": round(tr / cold / 1e9)}), flush=True)
    del mats
    torch.cuda.empty_cache()
'''

ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="sliced")
ap.add_argument("--configs", default="c2,c2f32,c2bf16,c1,c4")
ap.add_argument("--kinds", default="da")
ap.add_argument("--no-check", action="store_true", help="timing-only builds (results not exact)")
ap.add_argument("libs", nargs="+")
args = ap.parse_args()
for lib in args.libs:
    env = dict(os.environ)
    if lib != "base":
        env["DACSR_LIB_PATH"] = os.path.abspath(lib)
    tag = "base" if lib == "base" else os.path.basename(os.path.dirname(lib))
    for variant in args.variant.split(","):
        r = subprocess.run([sys.executable, "-c", CHILD, tag, variant, args.configs, args.kinds],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
        sys.stdout.write(r.stdout)
        if r.returncode:
            sys.stdout.write(f"# {tag} {variant} failed: {r.stderr[-1500:]}\n")
        sys.stdout.flush()
