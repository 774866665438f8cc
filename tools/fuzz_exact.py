"""Differential fuzz of the exact kernels against the CPU oracle (GPU box).

Random banded matrices (size, band, row-length law), both kinds, random row
ranges, alpha/beta and x_offset; every exact kernel and the default
selection must give the oracle's bits.  The fused group sums are checked
where they apply.

    python tools/fuzz_exact.py [seconds] [seed]
"""
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import numpy as np
import torch

import oracle
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.gen import banded_arrays, normal_vector
from paper_2307_06305_b200.power import chunk_partials, partials_from_groups

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
VERBOSE = len(sys.argv) > 3
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
dev = torch.device("cuda")
KERNELS = ("tiled", "sliced_pipe", "sliced", "wstream", "rowblock", "staged", "scalar")
t_end = time.time() + budget
cases = fails = 0
while time.time() < t_end:
    n = int(rng.choice([1, 33, 511, 512, 513, 4097, 20000, 70001, 150000]))
    b = int(rng.choice([1, 7, 300, 3000, 32767]))
    lam = float(rng.choice([0.3, 2.0, 8.0, 16.0, 40.0]))
    kmax = min(int(rng.choice([1, 4, 32, 64])), 2 * b + 1)  # kmax - 1 distinct offsets in [-b, b]
    seed = int(rng.integers(1, 1 << 30))
    print("case", n, b, lam, kmax, seed, flush=True)
    vdt = torch.float32 if rng.random() < 0.35 else torch.float64
    ndt = np.float32 if vdt == torch.float32 else np.float64
    bits_t = np.uint32 if vdt == torch.float32 else np.uint64
    arr = banded_arrays(n, b, lam, kmax, seed, dev, kinds=("da", "csr"), values_dtype=vdt)
    rp = arr["rowptr"].cpu().numpy()
    offs, cols, vals = (arr[k].cpu().numpy() for k in ("offsets", "colids", "values"))
    pad = int(rng.choice([0, 5, 64]))
    x = normal_vector(n, int(rng.integers(1, 1000)), dev).to(vdt)
    x_ext = torch.zeros(n + 2 * pad, dtype=vdt, device=dev)
    x_ext[pad:pad + n] = x
    xh = x.cpu().numpy()
    for kind, inner, ih in (("da", "offsets", offs), ("csr", "colids", cols)):
        dm = DeviceMatrix(kind, n, n, arr["rowptr"], arr[inner], arr["values"])
        for _ in range(2):
            r0, r1 = sorted(int(v) for v in rng.integers(0, n + 1, 2))
            if rng.random() < 0.3:
                r0, r1 = 0, n
            alpha, beta = [(1.0, 0.0), (0.7, -0.3), (2.0, 1.0), (-1.5, 0.5)][int(rng.integers(0, 4))]
            y0 = rng.uniform(-1, 1, n).astype(ndt)
            want = oracle.spmv_kernel(kind, rp, ih, vals, xh, y0.copy(), alpha, beta,
                                      row_start=r0, row_end=r1)
            for k in KERNELS + ("default",):
                y = torch.from_numpy(y0.copy()).to(dev)
                if VERBOSE:
                    print(" ", kind, k, r0, r1, alpha, beta, pad, flush=True)
                try:
                    if k == "default":
                        if (r0, r1) != (0, n) or pad:
                            continue
                        dg.spmv(dm, x, y, alpha, beta)
                    else:
                        xo = pad if kind == "da" else pad
                        dm.spmv_into(x_ext, y, alpha, beta, k, 0, x_offset=xo, row_start=r0,
                                     row_end=r1)
                except Exception as e:  # noqa: BLE001
                    if k in ("rowblock", "wstream") and (r0, r1) != (0, n):
                        continue  # planned for the whole range only
                    print("EXC", k, kind, n, b, lam, kmax, seed, r0, r1, repr(e)[:200], flush=True)
                    fails += 1
                    continue
                cases += 1
                torch.cuda.synchronize()
                if not np.array_equal(y.cpu().numpy().view(bits_t), want.view(bits_t)):
                    fails += 1
                    print("MISMATCH", k, kind, str(vdt), n, b, lam, kmax, seed, r0, r1, alpha, beta,
                          pad, flush=True)
        # fused group sums on whole-group ranges
        if kind == "da" and n >= 1024:
            dm.build_tiles()
            if dm.fused_sumsq_ok("tiled"):
                a_dev = torch.tensor([0.9], dtype=torch.float64, device=dev)
                gs = torch.empty((n + 511) // 512, dtype=torch.float64, device=dev)
                y = torch.empty(n, dtype=vdt, device=dev)
                dm.spmv_into(x, y, a_dev, 0.0, "tiled", 0, group_sumsq=gs)
                f = partials_from_groups(gs, n, 4096).cpu().numpy()
                d = chunk_partials(y, 4096).cpu().numpy()
                cases += 1
                if not np.array_equal(f.view(np.uint64), d.view(np.uint64)):
                    fails += 1
                    print("FUSED MISMATCH", n, b, lam, kmax, seed, flush=True)
    del arr, dm
print(f"cases {cases} failures {fails}", flush=True)
sys.exit(1 if fails else 0)
