"""Harness schema: records, serialisation, selection rule."""

import io

import numpy as np
import pytest

from paper_2307_06305_b200.model import StorageWidths
from paper_2307_06305_b200.suite import (BenchConfig, FormatSpec, ResultRecord, cache_bucket,
                                         materialize, verify, write_results)
from paper_2307_06305_b200.workloads import laplacian_2d


def _rec(**kw):
    base = dict(matrix_name="m", format="dacsr", oindex_bytes=4, iindex_bytes=2, scalar_bytes=8,
                variant="naive", threads=1, traffic_bytes=100, work_flops=10,
                time_seconds=0.1, performance_flops_per_s=100.0, throughput_bytes_per_s=1000.0,
                cache_bucket="HBM")
    base.update(kw)
    return ResultRecord(**base)


def test_csv_columns_follow_reference_then_gpu():
    buf = io.StringIO()
    write_results([_rec(best=True, kernel="wstream"), _rec(time_seconds=1 / 3)], buf)
    lines = buf.getvalue().splitlines()
    assert lines[0].split(",")[:14] == [
        "matrix_name", "format", "oindex_bytes", "iindex_bytes", "scalar_bytes", "variant",
        "threads", "traffic_bytes", "work_flops", "time_seconds", "performance_flops_per_s",
        "throughput_bytes_per_s", "cache_bucket", "best"]
    assert lines[0].endswith("kernel,cold")
    assert "true" in lines[1] and "0.33333333333333331" in lines[2]   # 17 significant digits
    js = io.StringIO()
    write_results([_rec()], js, format="json")
    assert '"kernel": ""' in js.getvalue()
    with pytest.raises(ValueError):
        write_results([], io.StringIO(), format="xml")


def test_config_and_format_validation():
    with pytest.raises(ValueError):
        BenchConfig(epochs=0)
    with pytest.raises(ValueError):
        FormatSpec("coo", StorageWidths(4, 4, 8))
    with pytest.raises(ValueError):
        FormatSpec("csr", StorageWidths(0, 4, 8))
    assert FormatSpec("dacsr", StorageWidths(4, 2, 8)).label == "dacsr(o32,i16,f64)"
    assert cache_bucket(126 << 20, 126 << 20) == "L2" and cache_bucket(1 + (126 << 20), 126 << 20) == "HBM"


def test_materialize_and_verify():
    a = laplacian_2d(16)
    d = materialize(a, FormatSpec("dacsr", StorageWidths(4, 1, 4)))
    assert d.colids.dtype == np.int8 and d.values.dtype == np.float32
    c = materialize(a, FormatSpec("csr", StorageWidths(8, 8, 8)))
    assert c.rowptr.dtype == np.int64 and c.colids.dtype == np.int64
    from paper_2307_06305_b200.errors import BandwidthExceedsIndexRange, IndexRangeExceeded
    with pytest.raises(BandwidthExceedsIndexRange):
        materialize(laplacian_2d(200), FormatSpec("dacsr", StorageWidths(4, 1, 8)))
    with pytest.raises(IndexRangeExceeded):
        materialize(laplacian_2d(200), FormatSpec("csr", StorageWidths(4, 1, 8)))
    ref = np.array([1.0, -2.0])
    assert verify(ref + 2 ** -42, ref, 8) and not verify(ref + 1e-9, ref, 8)
    assert verify(ref.astype(np.float32), ref, 4)


@pytest.mark.gpu
def test_run_suite_gpu(cuda):
    from paper_2307_06305_b200.suite import run_suite
    mats = [("lap", laplacian_2d(64)), ("wide", laplacian_2d(200))]
    fmts = [FormatSpec("csr", StorageWidths(4, 4, 8)), FormatSpec("dacsr", StorageWidths(4, 2, 8)),
            FormatSpec("dacsr", StorageWidths(4, 1, 8))]
    fake = iter(np.linspace(1e-3, 2e-3, 100).tolist())
    res = run_suite(mats, fmts, ["naive", "auto", "vector8"], BenchConfig(),
                    time_fn=lambda fn, cfg: next(fake))
    assert len(res.failures) == 1 and "BandwidthExceedsIndexRange" in res.failures[0].reason
    assert len(res.records) == 5 * 3
    for key in {(r.matrix_name, r.format, r.iindex_bytes) for r in res.records}:
        group = [r for r in res.records if (r.matrix_name, r.format, r.iindex_bytes) == key]
        best = [r for r in group if r.best]
        assert len(best) == 1 and best[0].time_seconds == min(r.time_seconds for r in group)
