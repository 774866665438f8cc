"""Generate the golden fixtures under tests/golden/ from the REFERENCE package.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [--c4]

Every output array here is produced by the reference's own code path
(`dacsr.spmv` with the numba backend, `dacsr.to_dacsr`, `dacsr.rcm`,
`dacsr.spmv.row_blocks`, `dacsr.model`), so the committed fixtures pin both
the oracle restatement (oracle/) and the CUDA path (through the oracle) to
the reference's behaviour.  Inputs are seeded and generated here.

Outputs:
  spmv_corpus.npz   random matrices (CSR i32 + DA i16/i8 + i64 rowptr cases),
                    x, y0, alpha, beta and the reference y of every serial
                    variant; csr==da and shifted_base==naive asserted here.
  conversions.npz   bandwidth / to_dacsr / to_csr boundary cases
  row_blocks.json   row_blocks(rowptr, k) cuts
  rcm.npz           reference rcm() permutations on small patterns, plus the
                    scrambled 256x256 Laplacian
  c4_rcm.json       (--c4) sha256 of reference rcm() on the scrambled
                    2048x2048 Laplacian (config C4), ~2 min of pure-Python BFS
  traffic.json      model.spmv_traffic / predicted_speedup values
"""

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF_SRC)

import dacsr  # noqa: E402  (the reference package)
from dacsr import generate as rgen  # noqa: E402
from dacsr.spmv import row_blocks as ref_row_blocks  # noqa: E402

VARIANTS = ("naive", "shifted_base", "multi_accumulator_3", "strip_mined_4")
AB = [(1.0, 0.0), (2.0, 0.5), (0.7, -0.3), (1.0, 1.0), (0.0, 1.0),
      (0.0, 0.0), (0.0, 2.5), (-1.25, 0.0), (3.0, -2.0)]
SEED = 20230711


def _ref_csr(nrows, ncols, rows, cols, vals, oindex=32, iindex=32, scalar=64):
    t = dacsr.TripletMatrix(nrows, ncols, rows, cols, vals)
    return dacsr.csr_from_triplets(t, oindex=oindex, iindex=iindex, scalar=scalar)


def _random_case(rng, i):
    nrows = int(rng.integers(0, 97)) if i % 23 else 0
    ncols = int(rng.integers(0, 97)) if i % 29 else 0
    if i % 7 == 3 and nrows:
        ncols = nrows
    density = float(rng.uniform(0.005, 0.45))
    scalar = 32 if i % 4 == 1 else 64
    target = int(round(density * nrows * ncols)) if nrows and ncols else 0
    rows = rng.integers(0, max(nrows, 1), target)
    cols = rng.integers(0, max(ncols, 1), target)
    vals = rng.uniform(-1.5, 1.5, target)
    vals[rng.random(target) < 0.05] = 0.0        # explicit zeros
    if target and i % 5 == 2:                      # duplicates (summed)
        k = max(1, target // 10)
        rows = np.concatenate([rows, rows[:k]])
        cols = np.concatenate([cols, cols[:k]])
        vals = np.concatenate([vals, rng.uniform(-1, 1, k)])
    oindex = 64 if i % 11 == 5 else 32
    return _ref_csr(nrows, ncols, rows, cols, vals, oindex=oindex, scalar=scalar)


def _special_cases(rng):
    out = []
    # paper Example-1 / reference conftest sample (4x4, 5 entries)
    s = [(0, 0, 1.0), (1, 2, 2.0), (2, 1, 3.0), (2, 3, 4.0), (3, 3, 5.0)]
    out.append(_ref_csr(4, 4, [e[0] for e in s], [e[1] for e in s], [e[2] for e in s]))
    # one long row (skew) among short rows
    n = 600
    rows = np.concatenate([np.arange(n), np.full(500, 17)])
    cols = np.concatenate([np.arange(n), rng.choice(n, 500, replace=False)])
    out.append(_ref_csr(n, n, rows, cols, rng.standard_normal(len(rows))))
    # all rows empty
    out.append(_ref_csr(7, 5, [], [], []))
    # single dense row / single dense column
    out.append(_ref_csr(1, 300, np.zeros(300, int), np.arange(300), rng.standard_normal(300)))
    out.append(_ref_csr(300, 1, np.arange(300), np.zeros(300, int), rng.standard_normal(300)))
    # banded, wide rows (vector-kernel territory)
    m = rgen.banded_random(400, 40, density=0.6, seed=3)
    out.append(m)
    # f32 banded
    out.append(rgen.banded_random(300, 12, density=0.5, seed=4, scalar=32))
    # tiny int8-width matrix (reference test_spmv.py:238-247)
    e = [(0, 0, 1.0), (1, 0, 2.0), (1, 2, 3.0), (3, 3, 4.0)]
    out.append(_ref_csr(4, 4, [a[0] for a in e], [a[1] for a in e], [a[2] for a in e],
                        oindex=8, iindex=8))
    return out


def make_spmv_corpus(n_random=200):
    rng = np.random.default_rng(SEED)
    mats = _special_cases(rng) + [_random_case(rng, i) for i in range(n_random)]
    data = {}
    meta = []
    for k, a in enumerate(mats):
        sd = a.values.dtype
        x = rng.uniform(-1.0, 1.0, a.ncols).astype(sd)
        alpha, beta = AB[k % len(AB)]
        if beta == 0.0:
            y0 = np.full(a.nrows, np.nan, dtype=sd)   # beta == 0 never reads y
        else:
            y0 = rng.uniform(-1.0, 1.0, a.nrows).astype(sd)
        try:
            iw = 8 if a.iindex_width == 8 else 16
            d = dacsr.to_dacsr(a, iw)
        except dacsr.errors.BandwidthExceedsIndexRange:
            d = dacsr.to_dacsr(a, 32)
        outs = {}
        for variant in VARIANTS:
            for m in (a, d):
                y = y0.copy()
                dacsr.spmv(m, x, y, alpha, beta, variant, backend="numba")
                outs.setdefault(variant, []).append(y)
        for variant in VARIANTS:
            yc, yd = outs[variant]
            assert np.array_equal(yc, yd, equal_nan=True), (k, variant)
        assert np.array_equal(outs["naive"][0], outs["shifted_base"][0], equal_nan=True)
        p = f"m{k}_"
        data[p + "rowptr"] = a.rowptr
        data[p + "colids"] = a.colids
        data[p + "offsets"] = d.colids
        data[p + "values"] = a.values
        data[p + "x"] = x
        data[p + "y0"] = y0
        data[p + "y_naive"] = outs["naive"][0]
        data[p + "y_macc3"] = outs["multi_accumulator_3"][0]
        data[p + "y_strip4"] = outs["strip_mined_4"][0]
        meta.append([a.nrows, a.ncols, alpha, beta])
    data["meta"] = np.array(meta, dtype=np.float64)
    data["count"] = np.array(len(mats))
    np.savez_compressed(os.path.join(HERE, "spmv_corpus.npz"), **data)
    print(f"spmv_corpus: {len(mats)} matrices")


def make_conversions():
    cases = []
    # (nrows, ncols, entries, iindex)
    cases.append((1, 2 ** 15, [(0, 2 ** 15 - 1, 1.0)], 16))      # w = 32767 fits
    cases.append((1, 2 ** 15 + 1, [(0, 2 ** 15, 1.0)], 16))      # w = 32768 rejected
    cases.append((1, 40001, [(0, 40000, 1.0)], 16))              # rejected
    cases.append((5, 5, [(4, 0, 2.0), (4, 4, 3.0)], 8))          # negative offsets
    cases.append((2, 10, [(0, 9, 1.0)], 16))                     # rectangular
    cases.append((6, 6, [(i, i, float(i + 1)) for i in range(6)], 8))
    cases.append((200, 200, [(i, (i * 37) % 200, 1.0) for i in range(200)], 8))  # 8-bit reject
    cases.append((0, 0, [], 16))
    rng = np.random.default_rng(11)
    for _ in range(20):
        nr, nc = int(rng.integers(1, 64)), int(rng.integers(1, 64))
        t = int(rng.integers(0, nr * nc // 4 + 1))
        ent = list(zip(rng.integers(0, nr, t).tolist(), rng.integers(0, nc, t).tolist(),
                       rng.uniform(0.5, 1.5, t).tolist()))
        cases.append((nr, nc, ent, 16))
    data = {}
    for k, (nr, nc, ent, iw) in enumerate(cases):
        a = _ref_csr(nr, nc, [e[0] for e in ent], [e[1] for e in ent], [e[2] for e in ent])
        p = f"c{k}_"
        data[p + "shape"] = np.array([nr, nc, iw])
        data[p + "rowptr"] = a.rowptr
        data[p + "colids"] = a.colids
        data[p + "values"] = a.values
        data[p + "bandwidth"] = np.array(dacsr.bandwidth(a))
        try:
            d = dacsr.to_dacsr(a, iw)
            data[p + "offsets"] = d.colids
            back = dacsr.to_csr(d, 32)
            assert back == a
            data[p + "ok"] = np.array(1)
        except dacsr.errors.BandwidthExceedsIndexRange:
            data[p + "ok"] = np.array(0)
    data["count"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "conversions.npz"), **data)
    print(f"conversions: {len(cases)} cases")


def make_row_blocks():
    rng = np.random.default_rng(5)
    out = []
    fixed = [[0, 1, 2, 4, 5, 9, 9, 12], [0, 0, 0, 0, 0, 0], [0], [0, 100], [0, 1, 1, 1, 50]]
    for rp in fixed:
        for k in (1, 2, 3, 7, 10):
            out.append({"rowptr": rp, "k": k,
                        "cuts": ref_row_blocks(np.array(rp, np.int64), k)})
    for _ in range(40):
        n = int(rng.integers(1, 60))
        rp = np.concatenate([[0], np.cumsum(rng.integers(0, 9, n))]).astype(np.int64)
        k = int(rng.integers(1, 12))
        out.append({"rowptr": rp.tolist(), "k": k, "cuts": ref_row_blocks(rp, k)})
    for item in out:
        item["cuts"] = [[int(a), int(b)] for a, b in item["cuts"]]
    with open(os.path.join(HERE, "row_blocks.json"), "w") as f:
        json.dump(out, f)
    print(f"row_blocks: {len(out)} cases")


def _laplacian_2d_ref(nx):
    """5-point Laplacian built independently through reference triplets."""
    idx = np.arange(nx * nx).reshape(nx, nx)
    rows, cols, vals = [idx.ravel()], [idx.ravel()], [np.full(nx * nx, 4.0)]
    for a, b in ((idx[1:, :], idx[:-1, :]), (idx[:, 1:], idx[:, :-1])):
        rows += [a.ravel(), b.ravel()]
        cols += [b.ravel(), a.ravel()]
        vals += [np.full(a.size, -1.0), np.full(a.size, -1.0)]
    return _ref_csr(nx * nx, nx * nx, np.concatenate(rows), np.concatenate(cols),
                    np.concatenate(vals))


def _sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr, dtype=np.int64).tobytes()).hexdigest()


def make_rcm():
    data = {}
    k = 0
    rng = np.random.default_rng(99)

    def add(a, tag):
        nonlocal k
        p = dacsr.rcm(a)
        pre = f"r{k}_"
        data[pre + "n"] = np.array(a.nrows)
        data[pre + "rowptr"] = a.rowptr.astype(np.int64)
        data[pre + "colids"] = a.colids.astype(np.int64)
        data[pre + "perm"] = p.perm
        b = dacsr.permute_symmetric(a, p)
        data[pre + "bw_after"] = np.array(dacsr.bandwidth(b))
        k += 1

    for i in range(40):  # acceptance crit-6 style: scrambled banded
        b = int(rng.integers(1, 33))
        n = int(rng.integers(max(3 * b, 20), 200))
        base = rgen.banded_random(n, b, density=float(rng.uniform(0.1, 0.5)), seed=1000 + i)
        mixed, _ = rgen.scrambled(base, seed=2000 + i)
        add(mixed, "banded")
    for i in range(25):  # random (unsymmetric, possibly disconnected) patterns
        n = int(rng.integers(1, 120))
        t = int(rng.integers(0, 3 * n + 1))
        a = _ref_csr(n, n, rng.integers(0, n, t), rng.integers(0, n, t), np.ones(t))
        add(a, "random")
    # diagonal-only, path, disconnected blocks
    add(_ref_csr(5, 5, range(5), range(5), np.ones(5)), "diag")
    e = [(0, 2), (2, 4), (4, 1), (1, 3)]
    r = [a for a, b in e] + [b for a, b in e]
    c = [b for a, b in e] + [a for a, b in e]
    add(_ref_csr(5, 5, r, c, np.ones(len(r))), "path")
    blocks = [rgen.banded_random(30, 3, seed=s) for s in range(3)]
    rows, cols, off = [], [], 0
    for bm in blocks:
        rr = np.repeat(np.arange(bm.nrows), np.diff(bm.rowptr))
        rows.append(rr + off)
        cols.append(bm.colids.astype(np.int64) + off)
        off += bm.nrows
    rr, cc = np.concatenate(rows), np.concatenate(cols)
    q = np.random.default_rng(1).permutation(off)
    add(_ref_csr(off, off, q[rr], q[cc], np.ones(len(rr))), "disconnected")
    # scrambled 256x256 Laplacian (n = 65536)
    lap = _laplacian_2d_ref(256)
    mixed, _ = rgen.scrambled(lap, seed=7)
    add(mixed, "laplace256")
    data["count"] = np.array(k)
    np.savez_compressed(os.path.join(HERE, "rcm.npz"), **data)
    print(f"rcm: {k} cases")


def make_c4():
    t0 = time.time()
    lap = _laplacian_2d_ref(2048)
    mixed, _ = rgen.scrambled(lap, seed=4)
    t1 = time.time()
    p = dacsr.rcm(mixed)
    t2 = time.time()
    after = dacsr.permute_symmetric(mixed, p)
    out = {
        "nx": 2048, "scramble_seed": 4,
        "laplacian_rowptr_sha256": _sha(lap.rowptr), "laplacian_colids_sha256": _sha(lap.colids),
        "scrambled_rowptr_sha256": _sha(mixed.rowptr),
        "scrambled_colids_sha256": _sha(mixed.colids),
        "perm_sha256": _sha(p.perm), "perm_head": p.perm[:16].tolist(),
        "bandwidth_scrambled": dacsr.bandwidth(mixed),
        "bandwidth_rcm": dacsr.bandwidth(after),
        "reference_rcm_seconds": round(t2 - t1, 1),
        "build_seconds": round(t1 - t0, 1),
    }
    with open(os.path.join(HERE, "c4_rcm.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("c4:", out)


def make_traffic():
    SW = dacsr.StorageWidths
    rows = []
    for n, nnz in [(1048576, 5238784), (2097152, 14581760), (2911419, 127729899),
                   (16777216, 268435456), (268435456, 2147483648), (4, 5), (0, 0)]:
        for w in [(4, 2, 8), (4, 4, 8), (4, 2, 4), (4, 4, 4), (8, 2, 8), (8, 4, 8), (4, 1, 8)]:
            t = dacsr.spmv_traffic(n, n, nnz, SW(*w))
            rows.append({"n": n, "nnz": nnz, "w": list(w), "total": t.total_bytes,
                         "rowptr": t.rowptr_bytes, "colids": t.colids_bytes,
                         "values": t.values_bytes, "vectors": t.vector_bytes})
    sp = dacsr.predicted_speedup(SW(4, 4, 8), SW(4, 2, 8), nrows=2097152, nnz=14581760)
    out = {"traffic": rows, "speedup_c2_f64": [sp.numerator, sp.denominator],
           "work_flops_bump": dacsr.work_flops(nnz=127729899, nrows=2911419)}
    with open(os.path.join(HERE, "traffic.json"), "w") as f:
        json.dump(out, f)
    print("traffic: ok")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--c4", action="store_true", help="also run reference rcm at C4 size")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    jobs = {"spmv": make_spmv_corpus, "conv": make_conversions, "rb": make_row_blocks,
            "rcm": make_rcm, "traffic": make_traffic}
    for name, fn in jobs.items():
        if not args.only or name in args.only.split(","):
            fn()
    if args.c4:
        make_c4()
