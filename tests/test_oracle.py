"""Pin the CPU oracle against fixtures the reference itself produced.

tests/golden/*.npz|json come from tests/golden/make_golden.py, which ran the
reference package (numba backend) in the build container.  If these pass,
the oracle is a bit-exact restatement of the reference on these inputs and
can serve as the checker for the CUDA path (tests/test_gpu_*.py).
"""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN

ORDER_KEYS = {"naive": "y_naive", "shifted_base": "y_naive",
              "multi_accumulator_3": "y_macc3", "strip_mined_4": "y_strip4"}


def load_corpus():
    z = np.load(os.path.join(GOLDEN, "spmv_corpus.npz"))
    cases = []
    for k in range(int(z["count"])):
        p = f"m{k}_"
        nrows, ncols, alpha, beta = z["meta"][k]
        cases.append(dict(
            nrows=int(nrows), ncols=int(ncols), alpha=alpha, beta=beta,
            **{name: z[p + name] for name in ("rowptr", "colids", "offsets", "values",
                                              "x", "y0", "y_naive", "y_macc3",
                                              "y_strip4")}))
    return cases


CORPUS = load_corpus()


def test_corpus_has_edge_cases():
    shapes = {(c["nrows"], c["ncols"]) for c in CORPUS}
    assert any(r == 0 for r, _ in shapes) and any(c == 0 for _, c in shapes)
    assert any(c["values"].dtype == np.float32 for c in CORPUS)
    assert any(c["rowptr"].dtype == np.int64 for c in CORPUS)
    assert any(c["offsets"].dtype == np.int8 for c in CORPUS)
    assert any(np.isnan(c["y0"]).any() for c in CORPUS)          # beta == 0 cases
    assert any(np.diff(c["rowptr"]).max(initial=0) >= 500 for c in CORPUS)


@pytest.mark.parametrize("variant", list(ORDER_KEYS))
@pytest.mark.parametrize("kind", ["csr", "da"])
def test_oracle_matches_reference_bit_exact(kind, variant):
    for k, c in enumerate(CORPUS):
        inner = c["colids"] if kind == "csr" else c["offsets"]
        y = c["y0"].copy()
        oracle.spmv(kind, c["rowptr"], inner, c["values"], c["x"], y, c["alpha"],
                    c["beta"], order=variant)
        want = c[ORDER_KEYS[variant]]
        assert np.array_equal(y.view(np.uint8), want.view(np.uint8)), (k, kind, variant)


@pytest.mark.parametrize("threads", [2, 3, 8])
def test_oracle_parallel_row_block_bit_identical(threads):
    for k, c in enumerate(CORPUS[:60]):
        if c["alpha"] == 0.0 or c["nrows"] == 0:
            continue
        y = c["y0"].copy()
        oracle.spmv("da", c["rowptr"], c["offsets"], c["values"], c["x"], y, c["alpha"],
                    c["beta"], order="naive", threads=threads)
        assert np.array_equal(y.view(np.uint8), c["y_naive"].view(np.uint8)), k


def test_row_blocks_golden():
    with open(os.path.join(GOLDEN, "row_blocks.json")) as f:
        cases = json.load(f)
    for c in cases:
        got = oracle.row_blocks(np.array(c["rowptr"], np.int64), c["k"])
        assert [list(b) for b in got] == c["cuts"], c


def test_conversions_golden():
    z = np.load(os.path.join(GOLDEN, "conversions.npz"))
    for k in range(int(z["count"])):
        p = f"c{k}_"
        nr, nc, iw = z[p + "shape"]
        rp, ci = z[p + "rowptr"], z[p + "colids"]
        assert oracle.bandwidth_csr(rp, ci) == int(z[p + "bandwidth"])
        off, ok = oracle.dacsr_offsets(rp, ci, int(iw))
        assert ok == bool(z[p + "ok"]), k
        if ok:
            assert off.dtype == z[p + "offsets"].dtype
            assert np.array_equal(off, z[p + "offsets"])


def test_rcm_golden():
    z = np.load(os.path.join(GOLDEN, "rcm.npz"))
    for k in range(int(z["count"])):
        p = f"r{k}_"
        n = int(z[p + "n"])
        perm = oracle.rcm(n, z[p + "rowptr"], z[p + "colids"])
        assert np.array_equal(perm, z[p + "perm"]), k


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def test_rcm_c4_hash():
    """Reference rcm() on the scrambled 2048² Laplacian (config C4, 92 s of
    pure-Python BFS when the fixture was made) reproduced by the oracle."""
    from paper_2307_06305_b200.workloads import laplacian_2d
    with open(os.path.join(GOLDEN, "c4_rcm.json")) as f:
        g = json.load(f)
    lap = laplacian_2d(g["nx"])
    assert _sha(lap.rowptr) == g["laplacian_rowptr_sha256"]
    assert _sha(lap.colids) == g["laplacian_colids_sha256"]
    n = lap.nrows
    order = np.random.default_rng(g["scramble_seed"]).permutation(n)
    rp, ci, _ = oracle.permute(n, lap.rowptr, lap.colids, lap.values, order)
    assert _sha(rp) == g["scrambled_rowptr_sha256"]
    assert _sha(ci) == g["scrambled_colids_sha256"]
    perm = oracle.rcm(n, rp, ci)
    assert _sha(perm) == g["perm_sha256"]


def test_traffic_golden():
    from paper_2307_06305_b200.model import StorageWidths, predicted_speedup, spmv_traffic
    with open(os.path.join(GOLDEN, "traffic.json")) as f:
        g = json.load(f)
    for row in g["traffic"]:
        t = spmv_traffic(row["n"], row["n"], row["nnz"], StorageWidths(*row["w"]))
        assert (t.total_bytes, t.rowptr_bytes, t.colids_bytes, t.values_bytes,
                t.vector_bytes) == (row["total"], row["rowptr"], row["colids"],
                                    row["values"], row["vectors"])
    sp = predicted_speedup(StorageWidths(4, 4, 8), StorageWidths(4, 2, 8),
                           nrows=2097152, nnz=14581760)
    assert [sp.numerator, sp.denominator] == g["speedup_c2_f64"]


def test_time_kernel_semantics():
    """bench.py:96-115: min over epochs of per-iteration time."""
    times = iter([0.0, 3.0, 10.0, 11.0, 20.0, 22.0])
    got = oracle.time_kernel(lambda: None, epochs=3, warmup_iters=0, min_epoch_iters=1,
                             min_epoch_time=0.0, clock=lambda: next(times))
    assert got == 1.0
