"""The 16-bit value extension of the CPU oracle (binary16 / bfloat16 values,
x and y; DeviceMatrix.astype on the GPU side), pinned without a GPU.

There is no reference kernel for 16-bit values (the reference stops at f32,
core.py:121-122); the contract is the one written in include/dacsr_b200.h:
f32 products of 16-bit significands are exact, the sum is f64 in the
reference's order, the epilogue alpha*acc (+ beta*y) is f64, one
round-to-nearest-even to 16 bits on the store.  These tests restate that in
pure Python (independent of the C oracle) and check both the conversions and
the kernels against it.
"""

import math

import numpy as np
import pytest

import oracle


def py_round16(d, bf16):
    """Pure-Python RNE of a float to binary16 / bfloat16 bits."""
    p, emin, ebias, emax = (8, -126, 127, 127) if bf16 else (11, -14, 15, 15)
    mb = p - 1
    sign = 0x8000 if math.copysign(1.0, d) < 0 else 0
    if math.isnan(d):
        return sign | ((2 * ebias + 1) << mb) | (1 << (mb - 1))
    a = abs(d)
    if a == 0.0:
        return sign
    if math.isinf(a):
        return sign | ((2 * ebias + 1) << mb)
    E = max(math.frexp(a)[1] - 1, emin)
    q = round(math.ldexp(a, mb - E))  # round-half-even on the exact float
    if q >= 1 << p:
        q >>= 1
        E += 1
    if E > emax:
        return sign | ((2 * ebias + 1) << mb)
    if q < 1 << mb:
        return sign | q
    return sign | ((E + ebias) << mb) | (q - (1 << mb))


def py_value16(b, bf16):
    return float(oracle.from_half_bits(np.array([b], np.uint16), bf16)[0])


@pytest.mark.parametrize("bf16", [False, True])
def test_half_conversions(bf16):
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.standard_normal(4000) * 10.0 ** rng.integers(-12, 12, 4000),
                        [0.0, -0.0, 65504.0, 65519.99, 65520.0, 5.96e-8, 2.98e-8, 2.99e-8,
                         3.39e38, 3.4e38, 1e-40, 9.2e-41, 60032.000930974384,
                         np.inf, -np.inf]])
    got = oracle.to_half_bits(x, bf16)
    want = np.array([py_round16(float(v), bf16) for v in x], np.uint16)
    assert np.array_equal(got, want)
    if not bf16:  # numpy rounds float64 -> float16 directly, RNE
        with np.errstate(over="ignore"):
            assert np.array_equal(got, x.astype(np.float16).view(np.uint16))
    # decoding is exact: re-rounding the decoded value is the identity
    back = oracle.from_half_bits(got, bf16)
    finite = np.isfinite(back)
    assert np.array_equal(oracle.to_half_bits(back[finite], bf16), got[finite])


def _py_spmv16(kind, rp, ci, vbits, xbits, ybits, alpha, beta, bf16, order):
    dec = lambda b: py_value16(int(b), bf16)  # noqa: E731
    out = ybits.copy()
    for r in range(len(rp) - 1):
        prods = []
        for i in range(rp[r], rp[r + 1]):
            c = ci[i] + (r if kind == "da" else 0)
            # exact product of two 16-bit significands (fits f32 and f64)
            prods.append(dec(vbits[i]) * dec(xbits[c]))
        if order == "naive":
            acc = 0.0
            for p_ in prods:
                acc += p_
        elif order == "multi_accumulator_3":
            a = [0.0, 0.0, 0.0]
            for k, p_ in enumerate(prods):
                a[k % 3] += p_
            acc = (a[0] + a[1]) + a[2]
        else:
            n4 = len(prods) // 4 * 4
            a = [0.0] * 4
            for k in range(n4):
                a[k % 4] += prods[k]
            acc = (a[0] + a[1]) + (a[2] + a[3])
            tail = 0.0
            for p_ in prods[n4:]:
                tail += p_
            acc = acc + tail
        t = alpha * acc if beta == 0.0 else alpha * acc + beta * dec(ybits[r])
        out[r] = py_round16(t, bf16)
    return out


@pytest.mark.parametrize("bf16", [False, True])
@pytest.mark.parametrize("kind", ["csr", "da"])
@pytest.mark.parametrize("order", ["naive", "multi_accumulator_3", "strip_mined_4"])
def test_half_kernels_match_python_restatement(bf16, kind, order):
    rng = np.random.default_rng(11)
    n = 120
    lens = rng.integers(0, 12, n)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    cols = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
    rows = np.repeat(np.arange(n), lens)
    ci = (cols - rows).astype(np.int16) if kind == "da" else cols.astype(np.int32)
    v = oracle.to_half_bits(rng.standard_normal(len(cols)), bf16)
    x = oracle.to_half_bits(rng.standard_normal(n) * 4, bf16)
    y0 = oracle.to_half_bits(rng.standard_normal(n), bf16)
    for alpha, beta in [(1.0, 0.0), (0.7, -0.3), (2.0, 0.5)]:
        want = _py_spmv16(kind, rp, ci, v, x, y0, alpha, beta, bf16, order)
        if bf16:
            y = y0.copy()
            oracle.spmv_kernel(kind, rp, ci, v, x, y, alpha, beta, order, bf16=True)
        else:
            y = y0.view(np.float16).copy()
            oracle.spmv_kernel(kind, rp, ci, v.view(np.float16), x.view(np.float16), y,
                               alpha, beta, order)
            y = y.view(np.uint16)
        assert np.array_equal(y, want), (alpha, beta)
