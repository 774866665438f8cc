"""TILED kernel probe (GPU box): bit-exactness on small wide-band matrices and
C3 / C5-slab timings against SLICED_PIPE.

    python tools/tiled_probe.py [--c3] [--c5rows N] [--tile-cols T]
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import numpy as np
import torch

import oracle
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.gen import banded_arrays, banded_device, normal_vector
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.model import StorageWidths, spmv_traffic

ap = argparse.ArgumentParser()
ap.add_argument("--c3", action="store_true")
ap.add_argument("--c5rows", type=int, default=0)
ap.add_argument("--tile-cols", type=int, default=None)
ap.add_argument("--kinds", default="da,csr")
args = ap.parse_args()
dev = torch.device("cuda")
out = {}


def small_checks():
    res = []
    for (n, b, lam, kmax, seed) in ((1 << 14, 3000, 16.0, 64, 5), (1 << 15, 32767, 8.0, 32, 6),
                                    (5000, 200, 30.0, 64, 7)):
        arr = banded_arrays(n, b, lam, kmax, seed, dev, kinds=("da", "csr"))
        rp = arr["rowptr"].cpu().numpy()
        x = normal_vector(n, 3, dev)
        xh = x.cpu().numpy()
        ref = oracle.spmv("da", rp, arr["offsets"].cpu().numpy(), arr["values"].cpu().numpy(), xh)
        for kind in ("da", "csr"):
            dm = DeviceMatrix(kind, n, n, arr["rowptr"], arr["offsets" if kind == "da" else "colids"],
                              arr["values"])
            for tc in (64, 256, 6144):
                dm.build_tiles(tc)
                y = torch.full((n,), 7.0, dtype=torch.float64, device=dev)
                dm.spmv_into(x, y, 1.0, 0.0, "tiled")
                ok = bool(np.array_equal(y.cpu().numpy().view(np.uint64), ref.view(np.uint64)))
                info = dm.tiles_info()
                res.append({"n": n, "b": b, "kind": kind, "tile_cols": tc, "exact": ok,
                            "n_ovf": info["n_ovf"]})
                # beta != 0, alpha != 1, row sub-range
                y0 = np.random.default_rng(1).uniform(-1, 1, n)
                y = torch.from_numpy(y0.copy()).to(dev)
                r0, r1 = n // 7, n - n // 5
                dm.spmv_into(x, y, 0.7, -0.3, "tiled", row_start=r0, row_end=r1)
                want = oracle.spmv_kernel("da", rp, arr["offsets"].cpu().numpy(),
                                          arr["values"].cpu().numpy(), xh, y0.copy(), 0.7, -0.3,
                                          row_start=r0, row_end=r1)
                ok2 = bool(np.array_equal(y.cpu().numpy().view(np.uint64), want.view(np.uint64)))
                res[-1]["exact_range_beta"] = ok2
    return res


out["small"] = small_checks()
print(json.dumps(out["small"]), flush=True)


def bench_pair(dm, x, label):
    o = dm.oindex_width // 8
    traffic = spmv_traffic(dm.nrows, dm.ncols, dm.nnz,
                           StorageWidths(o, dm.iindex_width // 8, dm.scalar_width // 8)).total_bytes
    r = {"bytes": traffic}
    t0 = time.time()
    dm.build_tiles(args.tile_cols)
    torch.cuda.synchronize()
    r["build_tiles_s"] = round(time.time() - t0, 2)
    r["tiles"] = dm.tiles_info()
    y1 = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dev)
    y2 = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dev)
    dm.spmv_into(x, y1, 1.0, 0.0, "tiled")
    dm.spmv_into(x, y2, 1.0, 0.0, "sliced_pipe")
    r["tiled_eq_sliced_pipe"] = bool(torch.equal(y1.view(torch.int64), y2.view(torch.int64)))
    for k in ("tiled", "sliced_pipe"):
        fn = lambda: dm.spmv_into(x, y1, 1.0, 0.0, k)
        warm = time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=3, min_epoch_time=0.0, graph=3)
        cold = time_kernel(fn, epochs=3, warmup_iters=1, min_epoch_iters=3, min_epoch_time=0.0, cold=True)
        r[k] = {"warm_us": round(warm * 1e6, 1), "cold_us": round(cold * 1e6, 1),
                "warm_gbs": round(traffic / warm / 1e9, 1), "cold_gbs": round(traffic / cold / 1e9, 1)}
    dm._sliced = None
    print(label, json.dumps(r), flush=True)
    return r


if args.c3:
    mats = banded_device("c3", dev, kinds=tuple(args.kinds.split(",")))
    x = normal_vector(mats["da" if "da" in mats else "csr"].ncols, 17, dev)
    for kind, dm in mats.items():
        out["c3_" + kind] = bench_pair(dm, x, "c3_" + kind)
if args.c5rows:
    from paper_2307_06305_b200.workloads import BANDED_CONFIGS
    n, b, lam, kmax, seed = BANDED_CONFIGS["c5"]
    arr = banded_arrays(n, b, lam, kmax, seed, dev, r0=0, r1=args.c5rows, kinds=("da",))
    dm = DeviceMatrix("da", args.c5rows, n, arr["rowptr"], arr["offsets"], arr["values"])
    x = normal_vector(n, 21, dev)
    out["c5slab"] = bench_pair(dm, x, "c5slab")
