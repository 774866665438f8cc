"""Benchmark: DA-CSR SpMV effective HBM GB/s on B200 vs the int32 CSR comparator.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0.  ``--impl reference`` times the reference's CPU path
(the oracle's C restatement of the reference kernels, ParallelRowBlock over
all host threads) on the same workload and prints the same line with
"impl": "reference".

Workload at N=1 (BASELINE.json configs[2], C3 — the largest configuration
that fits one GPU): random banded n = 2^24, half-bandwidth b = 32767, row
lengths clip(Poisson(16), 1, 64) with the diagonal, distinct uniform
offsets, values and x ~ N(0,1) (seeded counter-based generator, the same
rows on the device and in the CPU checker), DA-CSR with int16 offsets,
float64, int32 rowptr.  nnz = 268,211,692; the DA operator is 3.02 GB, far
beyond the 126 MB L2, which is additionally flushed before every step.  One
step = 100 back-to-back SpMVs y = A·x (one CUDA graph of 100 launches) with
the kernel the library's row-statistics selection picks for a plain
``spmv(A, x)`` (TILED for this matrix; no autotune).

value    = whole-job algorithmic GB/s = steps * 100 * spmv_traffic bytes / sum of
           step times (model.py / reference model.py:103-110: (n+1)*4 + nnz*(2+8)
           + 2n*8 bytes per SpMV)
e2e      = same metric through the public API spmv(A, x_host, y_host) with
           pinned host x / y (x H2D and y D2H inside every call; operator
           resident in HBM)
roofline = the dominant kernel (the selected exact kernel) vs the measured
           HBM copy peak in MEASURED_PEAKS.json

At N > 1 (torchrun) every rank runs config C5: 50 normalised power
iterations on the 2^28-row band, rows partitioned in contiguous blocks with
a +-b halo (distributed.py), strong scaling.
"""

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

SPMV_PER_STEP = 100
FALLBACK_HBM = 6650.0
READ_CEILING_GBS = 7268.4  # tools/peaks.py on this pool's B200 (profiles/ncu_summary.json)
METRIC = "SpMV effective HBM GB/s (DA-CSR i16, f64)"
C3_WORKLOAD = ("C3: random banded n=2^24, b=32767, clip(Poisson(16),1,64) with diagonal, "
               "N(0,1) values and x, DA-CSR i16 offsets + int32 rowptr, f64")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="naive")
    ap.add_argument("--no-suite", action="store_true", help="skip the other configs' lines")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--suite", default="c1,c2,c2xl,c2f32,c2bf16,c4,c5slab")
    ap.add_argument("--distributed", action="store_true",
                    help="run the N>1 (C5 power iteration, row blocks + halo) path at one rank")
    ap.add_argument("--workload", default="c3", choices=["c3", "c5"],
                    help="c3: 100 back-to-back SpMVs on C3 (default); "
                         "c5: 50-iteration power iteration on the 2^28-row band")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_key):
    """DRAM bytes per launch of the ncu --set full capture committed under
    profiles/ (ncu_summary.json), if present."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            rec = json.load(f).get(kernel_key, {})
        return rec.get("dram_bytes_per_launch"), rec
    except (OSError, ValueError):
        return None, {}


def traffic_of(n, nnz, o, i, s):
    from paper_2307_06305_b200.model import StorageWidths, spmv_traffic
    return spmv_traffic(n, n, nnz, StorageWidths(o, i, s)).total_bytes


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_mod():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    return oracle


def c3_host():
    """C3 on the host from the CPU checker's generator (the same rows as the
    device generator): rowptr i64, offsets i16, values f64, x f64."""
    from paper_2307_06305_b200.workloads import BANDED_CONFIGS, normal_table, poisson_cdf
    oracle = oracle_mod()
    n, b, lam, kmax, seed = BANDED_CONFIGS["c3"]
    table = normal_table()
    rp, offs, vals = oracle.gen_fill_parallel(n, b, kmax, seed, poisson_cdf(lam, kmax), table)
    x = oracle.gen_normal(17, 0, n, table)
    return n, rp, offs, vals, x


# ---------------------------------------------------------------- CPU leg
def cpu_measure(kind, rp, inner, vals, x, threads, budget_s=20.0):
    """The reference CPU path restated (oracle C port of _numba_kernels under
    ParallelRowBlock(threads)): best of the reference inner variants, each
    timed with the reference harness rule (min over epochs)."""
    oracle = oracle_mod()
    y = np.empty(len(rp) - 1, dtype=vals.dtype)
    best, best_var = math.inf, None
    t_start = time.perf_counter()
    for order in ("naive", "multi_accumulator_3", "strip_mined_4"):
        fn = lambda: oracle.spmv_kernel(kind, rp, inner, vals, x, y, 1.0, 0.0, order=order,
                                        threads=threads)
        t = oracle.time_kernel(fn, epochs=3, warmup_iters=1, min_epoch_iters=3,
                               min_epoch_time=0.1)
        if t < best:
            best, best_var = t, order
        if time.perf_counter() - t_start > budget_s:
            break
    return best, best_var


def numba_reference(rp, offs, vals, x, threads, rows, budget_s=25.0):
    """The reference package itself (numba kernels, ParallelRowBlock) from
    baseline/_ref, on the first ``rows`` rows, when it is installed there;
    None otherwise.  Seconds per SpMV of those rows."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "dacsr")):
        return None, "baseline/_ref not installed"
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_dacsr")
    sys.path.insert(0, ref_dir)
    try:
        import dacsr
        from dacsr.bench import BenchConfig, time_kernel
    except Exception as exc:  # numba missing on the host, etc.
        return None, f"import failed: {type(exc).__name__}: {exc}"
    e = int(rp[rows])
    a = dacsr.DacsrMatrix(rows, len(x), rp[:rows + 1].astype(np.int32), offs[:e], vals[:e])
    y = np.empty(rows)
    best, best_var = math.inf, None
    t0 = time.perf_counter()
    for inner in ("naive", "multi_accumulator_3", "strip_mined_4"):
        var = dacsr.ParallelRowBlock(threads, inner)
        fn = lambda: dacsr.spmv(a, x, y, 1.0, 0.0, var)
        t = time_kernel(fn, BenchConfig(epochs=3, warmup_iters=1, min_epoch_iters=3,
                                        min_epoch_time=0.1))
        if t < best:
            best, best_var = t, inner
        if time.perf_counter() - t0 > budget_s:
            break
    return (best, best_var), None


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    oracle = oracle_mod()
    threads = len(os.sched_getaffinity(0))
    n, rp, offs, vals, x = c3_host()
    traffic = traffic_of(n, len(offs), 4, 2, 8)
    t1, var = cpu_measure("da", rp, offs, vals, x, threads)
    # K timed steps of a bounded sample: SpMVs per step sized so the run ends
    # in about a minute (the metric is a rate)
    per_step = max(1, min(SPMV_PER_STEP, int(4.0 / max(t1, 1e-9))))
    y = np.empty(n)
    for _ in range(args.warmup):
        oracle.spmv_kernel("da", rp, offs, vals, x, y, 1.0, 0.0, order=var, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(per_step):
            oracle.spmv_kernel("da", rp, offs, vals, x, y, 1.0, 0.0, order=var,
                               threads=threads)
    el = time.perf_counter() - t0
    gbs = args.steps * per_step * traffic / el / 1e9
    sample = (f"C3 DA-CSR(i16) f64 (full matrix), {per_step} SpMVs per step, "
              f"ParallelRowBlock({threads}, '{var}') of the oracle C port; CPU {cpu_model()}")
    line = {
        "impl": "reference",
        "metric": METRIC, "value": round(gbs, 3),
        "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * el / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": C3_WORKLOAD, "spmv_per_step": per_step},
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU leg
def gpu_steps(fn_graph, steps, warmup, flush):
    """Per-step CUDA-event times (s) of a graph replay; L2 flushed before
    each step outside the events."""
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        flush()
        fn_graph()
    torch.cuda.synchronize()
    times = []
    for _ in range(steps):
        flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn_graph()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    return times


def measure_device(dm, x, variant, steps, warmup, per_step=SPMV_PER_STEP):
    """Graphed steps of ``per_step`` SpMVs with the kernel a plain spmv()
    call selects, plus the median of single cold SpMVs."""
    import torch
    from paper_2307_06305_b200.harness import GraphBatch, flush_l2
    from paper_2307_06305_b200.spmv import kernel_for, resolve_variant
    kname, order = resolve_variant(variant)
    kname = kernel_for(dm, kname, order)
    y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dm.device)
    dm.spmv_into(x, y, 1.0, 0.0, kname, order)  # builds the derived layout (once)
    torch.cuda.synchronize()
    g = GraphBatch(lambda: dm.spmv_into(x, y, 1.0, 0.0, kname, order), per_step)
    times = gpu_steps(g, steps, warmup, flush_l2)
    cold = []
    for _ in range(max(5, steps)):
        flush_l2()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        dm.spmv_into(x, y, 1.0, 0.0, kname, order)
        e1.record()
        e1.synchronize()
        cold.append(e0.elapsed_time(e1) / 1e3)
    del g
    return kname, order, times, sorted(cold)[len(cold) // 2], y


def measure_e2e(dm, x_host, steps, warmup, per_step):
    """Public API with pinned host buffers: every call copies x H2D and y
    D2H (pipelined by row pieces, hostpath.py); the operator stays in HBM."""
    import torch
    import paper_2307_06305_b200 as dg
    xp = torch.empty(len(x_host), dtype=torch.float64, pin_memory=True)
    xp.numpy()[:] = x_host
    yp = torch.empty(dm.nrows, dtype=torch.float64, pin_memory=True)
    xh, yh = xp.numpy(), yp.numpy()
    for _ in range(warmup):
        dg.spmv(dm, xh, yh)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        for _ in range(per_step):
            dg.spmv(dm, xh, yh)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps, yh


def suite_line(name, builder):
    """One config: DA and CSR, each with the default selection and with the
    fastest exact kernel (autotune), warm (graph of 10) and cold (L2
    flushed before each SpMV); the DA/CSR uplift against the traffic model."""
    import torch
    from paper_2307_06305_b200.harness import time_kernel
    from paper_2307_06305_b200.spmv import kernel_for
    t0 = time.time()
    mats, x, note = builder()
    out = {"build_s": round(time.time() - t0, 1), "note": note}
    for kind, dm in mats.items():
        o = dm.oindex_width // 8
        traffic = traffic_of(dm.nrows, dm.nnz, o, dm.iindex_width // 8, dm.scalar_width // 8)
        y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dm.device)
        rec = {"bytes": traffic, "nnz": dm.nnz}

        def warm_cold(k):
            fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, k, 0)
            fn()
            w = time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=2,
                            min_epoch_time=0.02, graph=10)
            c = time_kernel(fn, epochs=3, warmup_iters=1, min_epoch_iters=3,
                            min_epoch_time=0.0, cold=True)
            return w, c

        kdef = kernel_for(dm, "exact", 0)
        w, c = warm_cold(kdef)
        rec.update(kernel_default=kdef, warm_us=round(w * 1e6, 2), cold_us=round(c * 1e6, 2),
                   warm_gbs=round(traffic / w / 1e9, 1), cold_gbs=round(traffic / c / 1e9, 1))
        tuned = dm.autotune(x=x, reps=5)
        kbest = dm.tuned_kernel
        wb, cb = warm_cold(kbest)
        rec.update(kernel_tuned=kbest, tuned_warm_us=round(wb * 1e6, 2),
                   tuned_cold_us=round(cb * 1e6, 2),
                   autotune_warm_us={k: round(v * 1e6, 2) for k, v in tuned.items()},
                   default_over_tuned_cold=round(c / cb, 3))
        out[kind] = rec
    if "da" in out and "csr" in out:
        da, csr = out["da"], out["csr"]
        out["uplift_predicted"] = round(csr["bytes"] / da["bytes"], 4)
        out["uplift_default_cold"] = round(csr["cold_us"] / da["cold_us"], 4)
        out["uplift_best_cold"] = round(min(csr["cold_us"], csr["tuned_cold_us"]) /
                                        min(da["cold_us"], da["tuned_cold_us"]), 4)
        out["uplift_best_warm"] = round(min(csr["warm_us"], csr["tuned_warm_us"]) /
                                        min(da["warm_us"], da["tuned_warm_us"]), 4)
    del mats
    torch.cuda.empty_cache()
    return out


def suite_builders():
    import torch
    import paper_2307_06305_b200 as dg
    from paper_2307_06305_b200.device import DeviceMatrix
    from paper_2307_06305_b200.gen import banded_arrays, normal_vector
    from paper_2307_06305_b200.workloads import (BANDED_CONFIGS, laplacian_2d, laplacian_3d,
                                                 laplacian_3d_box, skewed_rcm_laplacian,
                                                 uniform_x)
    dev = torch.device("cuda")

    def host_pair(csr, x, note):
        return ({"da": DeviceMatrix.from_host(dg.to_dacsr(csr, 16)),
                 "csr": DeviceMatrix.from_host(csr)},
                torch.from_numpy(x).to(dev), note)

    def c1():
        csr = laplacian_2d(1024)
        return host_pair(csr, uniform_x(csr.ncols, 1), "2D 5-pt 1024^2 f64 (73 MB DA: L2-resident warm)")

    def c2():
        csr = laplacian_3d(128)
        return host_pair(csr, uniform_x(csr.ncols, 1), "3D 7-pt 128^3 f64 (188 MB DA)")

    def c2xl():
        # not a BASELINE config: C2's stencil and int16 offsets on a 1024 x 128 x 128
        # box, 8 times C2's rows — the stencil class well out of L2 (C2 itself
        # is a 36 us kernel of 1.5 x the L2 size)
        csr = laplacian_3d_box((1024, 128, 128))
        return host_pair(csr, uniform_x(csr.ncols, 1),
                         "3D 7-pt 1024x128x128 f64 (1.50 GB DA; C2's stencil out of L2, extension)")

    def c2f32():
        csr = laplacian_3d(128, np.float32)
        return host_pair(csr, uniform_x(csr.ncols, 1).astype(np.float32),
                         "3D 7-pt 128^3 f32 (113 MB DA)")

    def c2bf16():
        # width-lattice extension: bf16 values/x/y, f64 sums
        csr = laplacian_3d(128)
        mats = {k: DeviceMatrix.from_host(a).astype(torch.bfloat16)
                for k, a in (("da", dg.to_dacsr(csr, 16)), ("csr", csr))}
        x = torch.from_numpy(uniform_x(csr.ncols, 1)).to(dev).to(torch.bfloat16)
        return mats, x, "3D 7-pt 128^3 bf16 values/x/y, f64 accumulate (75 MB DA)"

    def c4():
        a, info = skewed_rcm_laplacian(2048)
        return host_pair(a, uniform_x(a.ncols, 1),
                         f"2048^2 Laplacian scrambled->RCM (w {info['bandwidth_scrambled']}->"
                         f"{info['bandwidth_rcm']}) + Pareto(1.5) skew rows, max row "
                         f"{int(np.diff(a.rowptr).max())}")

    def c5slab():
        # the first 2^25 rows of C5 (the full matrix is the N>1 workload)
        n, b, lam, kmax, seed = BANDED_CONFIGS["c5"]
        rows = 1 << 25
        arr = banded_arrays(n, b, lam, kmax, seed, dev, r0=0, r1=rows, kinds=("da", "csr"))
        mats = {"da": DeviceMatrix("da", rows, n, arr["rowptr"], arr["offsets"], arr["values"]),
                "csr": DeviceMatrix("csr", rows, n, arr["rowptr"], arr["colids"], arr["values"])}
        return mats, normal_vector(n, 21, dev), "C5 rows [0, 2^25): band b=32767, Poisson(8)"

    return {"c1": c1, "c2": c2, "c2xl": c2xl, "c2f32": c2f32, "c2bf16": c2bf16, "c4": c4,
            "c5slab": c5slab}


def measure_c5(steps, warmup, local=0):
    """Config C5 on one GPU: 50 normalised power iterations x <- A x / ||A x||
    on the 2^28-row band, DA-CSR i16, generated on the device, the 50
    iterations (SpMV with alpha read on the device, chunked norm, next alpha)
    captured once in a CUDA graph.  Returns (per-step seconds, record)."""
    import torch
    from paper_2307_06305_b200.device import DeviceMatrix
    from paper_2307_06305_b200.gen import banded_arrays, normal_vector
    from paper_2307_06305_b200.power import PowerIteration
    from paper_2307_06305_b200.spmv import kernel_for
    from paper_2307_06305_b200.workloads import BANDED_CONFIGS
    dev = torch.device("cuda", local)
    n, b, lam, kmax, seed = BANDED_CONFIGS["c5"]
    t0 = time.time()
    arr = banded_arrays(n, b, lam, kmax, seed, dev, kinds=("da",))
    dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"])
    x0 = normal_vector(n, 21, dev)
    build_s = time.time() - t0
    traffic = traffic_of(n, dm.nnz, dm.oindex_width // 8, 2, 8)
    iters = 50
    kname = kernel_for(dm, "exact", 0)
    pi = PowerIteration(dm, x0, iters=iters, variant=kname, graph=True)
    for _ in range(warmup):
        pi.run()
    torch.cuda.synchronize()
    times = []
    for _ in range(steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        pi.run()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    _, norms = pi.result()
    step = sum(times) / len(times)
    rec = {"workload": "C5: power iteration, 50 iters, banded n=2^28 b=32767 "
                       "clip(Poisson(8),1,32), DA-CSR i16",
           "value": round(iters * traffic / step / 1e9, 1), "unit": "GB/s",
           "ms_per_step": round(step * 1e3, 3), "steps": steps,
           "nnz": dm.nnz, "rowptr": str(dm.rowptr.dtype), "bytes_per_spmv": traffic,
           "build_s": round(build_s, 1), "final_norm": norms[-1], "kernel": kname,
           "cuda_graph": True}
    del pi, dm, arr
    torch.cuda.empty_cache()
    return times, rec


def run_c5(args, world, rank, local):
    """The C5 line at one GPU (``--workload c5``)."""
    import torch
    from paper_2307_06305_b200.harness import ClockSampler
    torch.cuda.set_device(local)
    with ClockSampler(local) as clocks:
        times, rec = measure_c5(args.steps, args.warmup, local)
    peak, peak_src = peaks()
    line = {
        "metric": METRIC, "value": rec["value"], "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {k: v for k, v in rec.items() if k not in ("value", "unit", "ms_per_step",
                                                            "steps")},
        "roofline": {"bound": "hbm", "achieved": rec["value"], "peak": peak, "unit": "GB/s",
                     "frac": round(rec["value"] / peak, 4), "traffic": None,
                     "peak_source": peak_src},
        "gpu_launches": args.steps * (50 * 3 + 3),
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import paper_2307_06305_b200 as dg
    from paper_2307_06305_b200.harness import ClockSampler

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.distributed:
        from paper_2307_06305_b200 import distributed
        return distributed.bench_main(args, rank, world, local)
    if args.workload == "c5":
        return run_c5(args, world, rank, local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2307_06305_b200.gen import banded_device, normal_vector

    t_build = time.time()
    mats = banded_device("c3", dev)
    dm, dmc = mats["da"], mats["csr"]
    x = normal_vector(dm.ncols, 17, dev)
    build_s = time.time() - t_build
    n, nnz = dm.nrows, dm.nnz
    t_da = traffic_of(n, nnz, 4, 2, 8)
    t_csr = traffic_of(n, nnz, 4, 4, 8)

    with ClockSampler(local) as clocks:
        kname, order, times, cold_da, y, = measure_device(dm, x, args.variant, args.steps,
                                                          args.warmup)
    step_s = sum(times) / len(times)
    value = SPMV_PER_STEP * t_da * len(times) / sum(times) / 1e9
    tiles = dm.tiles_info() if kname == "tiled" else None
    yh = y.cpu().numpy()
    kc, _, times_c, cold_csr, yc = measure_device(dmc, x, args.variant, max(3, args.steps // 2), 2)
    step_c = sum(times_c) / len(times_c)
    csr_equal = bool(torch.equal(yc, y))
    del yc
    dmc._tiled = dmc._sliced = None

    e2e_per = SPMV_PER_STEP // 10
    e2e_step, y_e2e = measure_e2e(dm, x.cpu().numpy(), max(2, args.steps // 5), 1, e2e_per)
    e2e_gbs = e2e_per * t_da / e2e_step / 1e9
    e2e_equal = bool(np.array_equal(y_e2e, yh))

    peak, peak_src = peaks()
    per_launch = step_s / SPMV_PER_STEP
    achieved = t_da / per_launch / 1e9
    traffic, ncu_rec = ncu_traffic(kname + ":c3:da")
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": C3_WORKLOAD, "n": n, "nnz": nnz, "bytes_per_spmv": t_da,
                   "spmv_per_step": SPMV_PER_STEP, "kernel": kname,
                   "kernel_selection": "library default for spmv(A, x): row statistics "
                                       "(dacsr_select_variant; gather scatter "
                                       f"{dm.stats.scatter:.3f}) -> {kname}; no autotune",
                   "layout": tiles,
                   "l2": "3.02 GB operator >> 126 MB L2; L2 flushed (read of 2x L2) before "
                         "every step",
                   "build_s": round(build_s, 1), "parallelism": "1 GPU"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_source": ncu_rec.get("source"),
                     "traffic_over_model": (round(traffic / t_da, 4) if traffic else None),
                     "dram_gbs_at_traffic": (round(traffic / per_launch / 1e9, 1)
                                             if traffic else None),
                     "peak_source": peak_src, "bytes_per_launch": t_da,
                     "frac_of_nominal_8TBs": round(achieved / 8000.0, 4),
                     "frac_of_tma_read_ceiling": round(achieved / READ_CEILING_GBS, 4),
                     "cold_single_spmv_gbs": round(t_da / cold_da / 1e9, 1)},
        "csr_comparator": {"kernel": kc, "value": round(SPMV_PER_STEP * t_csr / step_c / 1e9, 1),
                           "unit": "GB/s", "bytes_per_spmv": t_csr,
                           "uplift_measured": round(step_c / step_s, 4),
                           "uplift_measured_cold_single": round(cold_csr / cold_da, 4),
                           "uplift_predicted": round(t_csr / t_da, 4),
                           "y_bit_identical_to_da": csr_equal},
        "e2e": {"value": round(e2e_gbs, 1), "unit": "GB/s",
                "h2d_bytes_per_step": e2e_per * n * 8, "d2h_bytes_per_step": e2e_per * n * 8,
                "spmv_per_step": e2e_per, "y_bit_identical": e2e_equal,
                "note": "spmv(A, x_host, y_host) public API, pinned host x/y, operator "
                        "resident in HBM; PCIe-bound (256 MB of x + y cross per SpMV)"},
        "gflops": round(SPMV_PER_STEP * dg.work_flops(nnz=nnz, nrows=n) / step_s / 1e9, 1),
        "gpu_launches": args.steps * SPMV_PER_STEP,
        "clocks": clocks.summary(),
    }
    if not args.no_cpu:
        oracle = oracle_mod()
        threads = len(os.sched_getaffinity(0))
        rp = dm.rowptr.cpu().numpy()
        offs = dm.colids.cpu().numpy()
        vals = dm.values.cpu().numpy()
        xh = x.cpu().numpy()
        t_cpu, var = cpu_measure("da", rp, offs, vals, xh, threads)
        yref = oracle.spmv("da", rp, offs, vals, xh, threads=threads)
        line["parity_bit_exact_vs_oracle"] = bool(np.array_equal(yh.view(np.uint64),
                                                                 yref.view(np.uint64)))
        scaling = {}
        y_cpu = np.empty(n)
        for t in sorted({1, 4, threads}):
            fn = lambda t=t: oracle.spmv_kernel("da", rp, offs, vals, xh, y_cpu, 1.0, 0.0,
                                                order=var, threads=t)
            tt = oracle.time_kernel(fn, epochs=1, warmup_iters=0, min_epoch_iters=1,
                                    min_epoch_time=0.0)
            scaling[str(t)] = round(t_da / tt / 1e9, 2)
        ref_rows = 1 << 22
        numba_t, why = numba_reference(rp, offs, vals, xh, threads, ref_rows)
        t_ref_rows = traffic_of(ref_rows, int(rp[ref_rows]), 4, 2, 8)
        line["cpu_baseline"] = {
            "value": round(t_da / t_cpu / 1e9, 3), "unit": "GB/s", "cores": threads,
            "gbs_by_threads": scaling, "kind": "port",
            "sample": f"C3 DA-CSR f64 (full matrix), one SpMV per iteration, best of the "
                      f"reference inner variants ('{var}' won) under ParallelRowBlock({threads}),"
                      f" 3 epochs of >=3 iters/>=0.1 s; oracle C port of _numba_kernels; "
                      f"CPU {cpu_model()}",
            "reference_numba": (
                {"value": round(t_ref_rows / numba_t[0] / 1e9, 3), "unit": "GB/s",
                 "kind": "reference", "cores": threads,
                 "sample": f"the reference package itself (baseline/_ref, numba) "
                           f"spmv(DacsrMatrix, x, y, 1, 0, ParallelRowBlock({threads}, "
                           f"'{numba_t[1]}')) on C3 rows [0, 2^22), reference time_kernel"}
                if numba_t else {"unavailable": why})}
    del dm, dmc, mats
    torch.cuda.empty_cache()
    if not args.no_suite:
        # config C5 at one GPU: the base of the N>1 strong-scaling runs
        # (bench.py --gpus N runs the same 50 iterations over N ranks)
        try:
            _, line["c5_power_iteration_1gpu"] = measure_c5(3, 1, local)
        except Exception as exc:
            line["c5_power_iteration_1gpu"] = {"error": f"{type(exc).__name__}: {exc}"}
        suite = {}
        builders = suite_builders()
        for name in args.suite.split(","):
            if name in builders:
                try:
                    suite[name] = suite_line(name, builders[name])
                except Exception as exc:  # a suite line must not sink the headline
                    suite[name] = {"error": f"{type(exc).__name__}: {exc}"}
        line["suite"] = suite
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
