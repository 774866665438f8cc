"""``python -m paper_2307_06305_b200 bench`` — the GPU counterpart of the
reference's ``dacsr bench`` (cli.py:215-283) for the BASELINE configs.

    python -m paper_2307_06305_b200 bench --generate c1,c2 --formats csr,dacsr \
        --variants naive,auto --out results.csv

Prints the reference's table (matrix, format, variant, threads, time,
GFLOP/s, GB/s, bucket, best) and the "best dacsr vs best csr" line, and
writes the records with ``suite.write_results``.  Exit codes follow the
reference: 0 ok, 1 nothing measured, 2 usage error.
"""

import argparse
import sys

import numpy as np


def _matrices(spec):
    from .workloads import laplacian_2d, laplacian_3d, skewed_rcm_laplacian
    for name in spec.split(","):
        name = name.strip()
        if name == "c1":
            yield "c1-laplace2d-1024", laplacian_2d(1024)
        elif name == "c2":
            yield "c2-laplace3d-128", laplacian_3d(128)
        elif name == "c4":
            yield "c4-rcm-skew-2048", skewed_rcm_laplacian(2048)[0]
        elif name.startswith("lap2d:"):
            n = int(name.split(":")[1])
            yield f"laplace2d-{n}", laplacian_2d(n)
        else:
            raise ValueError(f"unknown matrix spec {name!r} (c1, c2, c4, lap2d:N)")


def _table(rows, headers, fh):
    widths = [max(len(str(h)), *(len(str(r[i])) for r in rows)) for i, h in enumerate(headers)]
    fh.write("  ".join(str(h).ljust(w) for h, w in zip(headers, widths)) + "\n")
    for r in rows:
        fh.write("  ".join(str(c).ljust(w) for c, w in zip(r, widths)) + "\n")


def cmd_bench(args):
    from .model import StorageWidths, relative_performance
    from .suite import BenchConfig, FormatSpec, run_suite, write_results
    formats = []
    for kind in args.formats.split(","):
        kind = kind.strip()
        ib = args.csr_iindex if kind == "csr" else args.dacsr_iindex
        if kind not in ("csr", "dacsr"):
            print(f"error: unknown format {kind!r}", file=sys.stderr)
            return 2
        formats.append(FormatSpec(kind, StorageWidths(args.oindex // 8, ib // 8,
                                                      args.scalar // 8)))
    cfg = BenchConfig(epochs=args.epochs, warmup_iters=args.warmup,
                      min_epoch_iters=args.min_epoch_iters,
                      min_epoch_time=args.min_epoch_ms / 1000.0, cold=args.cold)
    variants = [v.strip() for v in args.variants.split(",") if v.strip()]
    try:
        mats = list(_matrices(args.generate))
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    suite = run_suite(mats, formats, variants, cfg, seed=args.seed)
    for f in suite.failures:
        print(f"skipped: {f.matrix_name} [{f.format}]: {f.reason}", file=sys.stderr)
    rows = [[r.matrix_name, r.format, r.variant, r.kernel, r.threads,
             f"{r.time_seconds:.3e}", f"{r.performance_flops_per_s / 1e9:.3f}",
             f"{r.throughput_bytes_per_s / 1e9:.3f}", r.cache_bucket, "*" if r.best else ""]
            for r in suite.records]
    _table(rows, ["matrix", "format", "variant", "kernel", "threads", "time_s", "gflop_per_s",
                  "gbyte_per_s", "bucket", "best"], sys.stdout)
    best = {(r.matrix_name, r.format): r for r in suite.records if r.best}
    for name in dict.fromkeys(n for n, _ in best):
        c, d = best.get((name, "csr")), best.get((name, "dacsr"))
        if c and d:
            print(f"{name}: best dacsr vs best csr performance: "
                  f"{relative_performance(c.time_seconds, d.time_seconds):.3f}x")
    if args.out:
        write_results(suite.records, args.out, format="json" if args.json else "csv")
    return 0 if suite.records else 1


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2307_06305_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="time SpMV formats/variants on the GPU")
    b.add_argument("--generate", default="c1,c2")
    b.add_argument("--formats", default="csr,dacsr")
    b.add_argument("--variants", default="naive")
    b.add_argument("--oindex", type=int, default=32)
    b.add_argument("--csr-iindex", type=int, default=32)
    b.add_argument("--dacsr-iindex", type=int, default=16)
    b.add_argument("--scalar", type=int, default=64)
    b.add_argument("--epochs", type=int, default=11)
    b.add_argument("--warmup", type=int, default=10)
    b.add_argument("--min-epoch-iters", type=int, default=10)
    b.add_argument("--min-epoch-ms", type=float, default=100.0)
    b.add_argument("--cold", action="store_true", help="flush L2 before every timed SpMV")
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--out")
    b.add_argument("--json", action="store_true")
    args = ap.parse_args(argv)
    if args.cmd == "bench":
        return cmd_bench(args)
    return 2


if __name__ == "__main__":
    sys.exit(main())
