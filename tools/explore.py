"""Scratch GPU exploration: GB/s of every variant on the BASELINE configs."""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.gen import banded_device, normal_vector
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.model import StorageWidths, spmv_traffic
from paper_2307_06305_b200.workloads import laplacian_2d, laplacian_3d, uniform_x

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2,c2f32,c3")
ap.add_argument("--variants", default="naive,wstream,rowblock,scalar,vector4,vector8")
ap.add_argument("--cold", action="store_true")
args = ap.parse_args()
dev = torch.device("cuda")
out = []


def run(name, mats, x):
    for kind, dm in mats.items():
        o = dm.oindex_width // 8
        tr = spmv_traffic(dm.nrows, dm.ncols, dm.nnz, StorageWidths(o, dm.iindex_width // 8,
                                                                   dm.scalar_width // 8)).total_bytes
        y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dev)
        for v in args.variants.split(","):
            from paper_2307_06305_b200.spmv import kernel_for, resolve_variant
            kname, order = resolve_variant(v)
            kname = kernel_for(dm, kname, order)
            fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, kname, order)
            try:
                t = time_kernel(fn, epochs=5, warmup_iters=3, min_epoch_iters=3,
                                min_epoch_time=0.05, cold=args.cold, graph=0 if args.cold else 20)
            except Exception as e:  # noqa
                print(name, kind, v, "ERROR", e, flush=True)
                continue
            if kname == "wstream":
                v += f"[vcap={dm.chunk_plan().chunk_vcap},cx={dm.chunk_plan().n_complex}]"
            if kname == "sliced":
                inf = dm.slices_info()
                v += f"[T={inf['max_len']},pad={inf['padding']:.3f},med={inf['n_medium']},long={inf['n_long']}]"
            rec = dict(config=name, kind=kind, variant=v, us=t * 1e6, gbs=tr / t / 1e9,
                       bytes=tr, cold=args.cold, plan_cap=dm.plan.cap if dm.plan else None)
            out.append(rec)
            print(json.dumps(rec), flush=True)


for c in args.configs.split(","):
    t0 = time.time()
    if c == "c2bf16":
        csr = laplacian_3d(128)
        mats = {k: DeviceMatrix.from_host(a).astype(torch.bfloat16)
                for k, a in (("csr", csr), ("da", dg.to_dacsr(csr, 16)))}
        x = torch.from_numpy(uniform_x(csr.ncols, 1)).to(dev).to(torch.bfloat16)
    elif c in ("c1", "c2", "c2f32"):
        dt = np.float32 if c == "c2f32" else np.float64
        csr = laplacian_2d(1024, dt) if c == "c1" else laplacian_3d(128, dt)
        mats = {"csr": DeviceMatrix.from_host(csr), "da": DeviceMatrix.from_host(dg.to_dacsr(csr, 16))}
        x = torch.from_numpy(uniform_x(csr.ncols, 1).astype(dt)).to(dev)
    elif c == "c3":
        mats = banded_device("c3", dev)
        x = normal_vector(mats["da"].ncols, 17, dev)
    elif c == "c4":
        from paper_2307_06305_b200.workloads import skewed_rcm_laplacian
        a, info = skewed_rcm_laplacian(2048)
        mats = {"csr": DeviceMatrix.from_host(a), "da": DeviceMatrix.from_host(dg.to_dacsr(a, 16))}
        x = torch.from_numpy(uniform_x(a.ncols, 1)).to(dev)
        st = mats["da"].stats
        print(f"# c4 stats mean {st.mean_len:.2f} max {st.max_len} cv {st.cv_len:.2f}; "
              f"complex chunks (256) {mats['da'].chunk_plan(256).n_complex}", flush=True)
    print(f"# {c} built in {time.time()-t0:.1f}s", flush=True)
    run(c, mats, x)
    del mats
    torch.cuda.empty_cache()
