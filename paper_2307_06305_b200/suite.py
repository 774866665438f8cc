"""GPU benchmark suite in the reference harness's schema.

Same records and selection rule as the reference's ``run_suite``
(/root/reference/pkg/src/dacsr/bench.py:160-238) and ``ResultRecord`` /
``write_results`` (io.py:28-46, 183-215), so GPU and CPU results land in the
same CSV/JSON columns:

* every (matrix, format, variant) is materialised at the format's widths,
  run once and verified against naive CSR at 64-bit widths with the
  reference tolerance (2^-40 f64, 1e-5 f32, relative to max|ref|), then
  timed with the warm-up / epoch / best-of rule — on the device, with CUDA
  events (``harness.time_kernel``);
* conversion or verification failures are recorded, never fatal;
* the highest-performance record per (matrix, format) carries ``best``.

GPU-specific: ``threads`` is 1 (one device), ``cache_bucket`` is "L2" when
the SpMV's traffic fits the device L2 and "HBM" otherwise, and the extra
columns ``kernel`` (the launched kernel) and ``cold`` (L2 flushed before each
timed SpMV) follow the reference's columns.
"""

import csv
import dataclasses
import json
from dataclasses import dataclass, field

import numpy as np

from .core import CsrMatrix, index_max, scalar_dtype, to_dacsr, _trusted
from .errors import DacsrError, IndexRangeExceeded
from .model import StorageWidths, spmv_traffic
from .spmv import work_flops


@dataclass(frozen=True)
class BenchConfig:
    """Timing rule of the reference (bench.py:27-43)."""

    epochs: int = 11
    warmup_iters: int = 10
    min_epoch_iters: int = 10
    min_epoch_time: float = 0.1
    cold: bool = False

    def __post_init__(self):
        if self.epochs < 1:
            raise ValueError("epochs must be >= 1")
        if self.min_epoch_time < 0:
            raise ValueError("min_epoch_time must be >= 0")
        if self.warmup_iters < 0 or self.min_epoch_iters < 0:
            raise ValueError("warmup_iters and min_epoch_iters must be >= 0")


@dataclass(frozen=True)
class FormatSpec:
    """A storage format to benchmark: "csr" or "dacsr" at given widths."""

    kind: str
    widths: StorageWidths

    def __post_init__(self):
        if self.kind not in ("csr", "dacsr"):
            raise ValueError(f"kind must be csr or dacsr, got {self.kind!r}")
        if self.widths.oindex_bytes == 0 or self.widths.iindex_bytes == 0:
            raise ValueError("benchmark formats need physical index widths")

    @property
    def label(self):
        w = self.widths
        return f"{self.kind}(o{w.oindex_bytes * 8},i{w.iindex_bytes * 8},f{w.scalar_bytes * 8})"


@dataclass
class ResultRecord:
    """One timed run; columns of the reference's ResultRecord, then GPU ones."""

    matrix_name: str
    format: str
    oindex_bytes: int
    iindex_bytes: int
    scalar_bytes: int
    variant: str
    threads: int
    traffic_bytes: int
    work_flops: int
    time_seconds: float
    performance_flops_per_s: float
    throughput_bytes_per_s: float
    cache_bucket: str
    best: bool = False
    kernel: str = ""
    cold: bool = False


@dataclass
class ConversionFailure:
    matrix_name: str
    format: str
    reason: str


@dataclass
class SuiteResult:
    records: list = field(default_factory=list)
    failures: list = field(default_factory=list)


def cache_bucket(traffic_bytes, l2_bytes):
    """"L2" when one SpMV's traffic fits the device L2, else "HBM"."""
    return "L2" if traffic_bytes <= l2_bytes else "HBM"


def materialize(base, fmt):
    """Re-store ``base`` at ``fmt``'s widths with the reference's range checks
    (bench.py:129-150)."""
    w = fmt.widths
    obits, ibits = w.oindex_bytes * 8, w.iindex_bytes * 8
    if base.nnz > index_max(obits):
        raise IndexRangeExceeded(f"nnz = {base.nnz} does not fit o{obits}")
    rowptr = base.rowptr.astype(np.dtype(f"int{obits}"))
    values = base.values.astype(scalar_dtype(w.scalar_bytes * 8))
    if fmt.kind == "csr":
        if base.ncols > 0 and base.ncols - 1 > index_max(ibits):
            raise IndexRangeExceeded(f"ncols = {base.ncols} does not fit i{ibits}")
        return _trusted(CsrMatrix, base.nrows, base.ncols, rowptr,
                        base.colids.astype(np.dtype(f"int{ibits}")), values)
    wide = _trusted(CsrMatrix, base.nrows, base.ncols, rowptr, base.colids.astype(np.int64),
                    values)
    return to_dacsr(wide, ibits)


def verify(y, ref, scalar_bytes):
    """The reference's acceptance rule (bench.py:153-157)."""
    tol = 2.0 ** -40 if scalar_bytes == 8 else 1e-5
    scale = max(float(np.max(np.abs(ref))) if len(ref) else 0.0, 1e-30)
    err = float(np.max(np.abs(np.asarray(y, np.float64) - ref))) if len(ref) else 0.0
    return err <= tol * scale


def run_suite(matrices, formats, variants, cfg, seed=0, time_fn=None, device=None):
    """Benchmark every (matrix, format, variant) on the GPU."""
    import torch

    from .device import DeviceMatrix
    from .harness import l2_bytes, time_kernel
    from .spmv import kernel_for, resolve_variant

    device = torch.device(device or "cuda")
    l2 = l2_bytes(device)
    rng = np.random.default_rng(seed)
    out = SuiteResult()
    for name, base in matrices:
        x64 = rng.uniform(0.5, 1.5, base.ncols)
        refs = {}
        for fmt in formats:
            try:
                mat = materialize(base, fmt)
            except DacsrError as exc:
                out.failures.append(ConversionFailure(name, fmt.label,
                                                      f"{type(exc).__name__}: {exc}"))
                continue
            sb = fmt.widths.scalar_bytes
            xt = torch.from_numpy(x64.astype(scalar_dtype(sb * 8))).to(device)
            if sb not in refs:
                ref_mat = materialize(base, FormatSpec("csr", StorageWidths(8, 8, sb)))
                dref = DeviceMatrix.from_host(ref_mat, device)
                yref = torch.empty(base.nrows, dtype=xt.dtype, device=device)
                dref.spmv_into(xt, yref, 1.0, 0.0, "scalar", 0)
                refs[sb] = yref.cpu().numpy().astype(np.float64)
            ref = refs[sb]
            dm = DeviceMatrix.from_host(mat, device)
            traffic = spmv_traffic(base.nrows, base.ncols, base.nnz, fmt.widths).total_bytes
            work = work_flops(base)
            recs = []
            for variant in variants:
                kname, order = resolve_variant(variant)
                kname = kernel_for(dm, kname, order)
                y = torch.empty(base.nrows, dtype=xt.dtype, device=device)
                fn = lambda dm=dm, y=y, k=kname, o=order: dm.spmv_into(xt, y, 1.0, 0.0, k, o)
                fn()
                if not verify(y.cpu().numpy(), ref, sb):
                    out.failures.append(ConversionFailure(
                        name, fmt.label, f"verification failed for {variant} ({kname})"))
                    continue
                if time_fn is not None:
                    secs = time_fn(fn, cfg)
                else:
                    secs = time_kernel(fn, epochs=cfg.epochs, warmup_iters=cfg.warmup_iters,
                                       min_epoch_iters=cfg.min_epoch_iters,
                                       min_epoch_time=cfg.min_epoch_time, cold=cfg.cold,
                                       graph=0 if cfg.cold else 10)
                recs.append(ResultRecord(
                    matrix_name=name, format=fmt.kind, oindex_bytes=fmt.widths.oindex_bytes,
                    iindex_bytes=fmt.widths.iindex_bytes, scalar_bytes=sb, variant=str(variant),
                    threads=1, traffic_bytes=traffic, work_flops=work, time_seconds=secs,
                    performance_flops_per_s=work / secs, throughput_bytes_per_s=traffic / secs,
                    cache_bucket=cache_bucket(traffic, l2), kernel=kname, cold=cfg.cold))
            if recs:
                max(recs, key=lambda r: r.performance_flops_per_s).best = True
                out.records.extend(recs)
    return out


def _cell(v):
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        return f"{v:.17g}"
    return v


def write_results(records, sink, format="csv"):
    """CSV (fixed header, record field order, 17 significant digits) or a
    JSON array — the reference's serialisation (io.py:191-215)."""
    if format not in ("csv", "json"):
        raise ValueError(f"format must be csv or json, got {format!r}")
    names = [f.name for f in dataclasses.fields(ResultRecord)]

    def emit(fh):
        if format == "csv":
            w = csv.writer(fh, lineterminator="\n")
            w.writerow(names)
            for r in records:
                w.writerow([_cell(getattr(r, n)) for n in names])
        else:
            json.dump([dataclasses.asdict(r) for r in records], fh, indent=2)
            fh.write("\n")

    if hasattr(sink, "write"):
        emit(sink)
    else:
        with open(sink, "w", encoding="utf-8", newline="") as fh:
            emit(fh)


__all__ = ["BenchConfig", "ConversionFailure", "FormatSpec", "ResultRecord", "SuiteResult",
           "cache_bucket", "materialize", "run_suite", "verify", "write_results"]
