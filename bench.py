"""Benchmark: DA-CSR SpMV effective HBM GB/s on B200 vs the int32 CSR comparator.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0.  ``--impl reference`` times the reference's CPU path
(the oracle's C restatement of the reference kernels, ParallelRowBlock over
all host threads) on the same workload and prints the same line with
"impl": "reference".

Workload (BASELINE.json configs[1], C2): 3D 7-point Laplacian on a 128^3
grid, n = 2,097,152, nnz = 14,581,760, float64, DA-CSR with int16 offsets
(bandwidth 16384), x ~ U[-1,1] (seed 1).  One step = 100 back-to-back
SpMVs y = A·x (one CUDA graph of 100 launches).  The DA matrix is 188 MB
(> the 126 MB L2) and L2 is additionally flushed (a read of 2x L2, which
leaves clean lines) before every step, outside the step's CUDA events.

value    = whole-job algorithmic GB/s = steps * 100 * spmv_traffic bytes / sum of
           step times (model.py / reference model.py:103-110: (n+1)*4 + nnz*(2+8)
           + 2n*8 bytes per SpMV)
e2e      = same metric through the public API spmv(A, x_host, y_host) with
           pinned host x/y: every SpMV copies x H2D and y D2H inside the step
roofline = the dominant kernel (the selected exact kernel) vs the measured
           HBM copy peak in MEASURED_PEAKS.json
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="naive")
    ap.add_argument("--no-suite", action="store_true", help="skip the C1/C2-f32/C3/C4 lines")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--suite", default="c1,c2f32,c2bf16,c3,c4")
    ap.add_argument("--distributed", action="store_true",
                    help="use the row-block/halo path even at one rank (plumbing check)")
    ap.add_argument("--workload", default="c2", choices=["c2", "c5"],
                    help="c2: 100 back-to-back SpMVs (default); c5: 50-iteration power "
                         "iteration on the 2^28-row banded matrix")
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
    """(dram bytes per cold launch from the ncu --set full capture, the
    steady-state record inside the bench step) from the committed ncu
    summary, if present."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            rec = json.load(f).get(kernel_key, {})
        return rec.get("dram_bytes_per_launch"), rec.get("steady_state_in_step")
    except (OSError, ValueError):
        return None, None


def c2_host(dtype=np.float64):
    import paper_2307_06305_b200 as dg
    from paper_2307_06305_b200.workloads import laplacian_3d, uniform_x
    csr = laplacian_3d(128, dtype)
    return csr, dg.to_dacsr(csr, 16), uniform_x(csr.ncols, seed=1).astype(dtype)


def traffic_of(n, nnz, o, i, s):
    from paper_2307_06305_b200.model import StorageWidths, spmv_traffic
    return spmv_traffic(n, n, nnz, StorageWidths(o, i, s)).total_bytes


# ---------------------------------------------------------------- CPU leg
def cpu_measure(kind, a, x, threads, budget_s=20.0):
    """Reference CPU path (oracle C port of the reference kernels) on the
    host: best of the reference inner variants under ParallelRowBlock."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    y = np.empty(a.nrows, dtype=a.values.dtype)
    best = math.inf
    best_var = None
    t_start = time.perf_counter()
    for order in ("naive", "multi_accumulator_3", "strip_mined_4"):
        fn = lambda: oracle.spmv_kernel(kind, a.rowptr, a.colids, a.values, x, y, 1.0, 0.0,
                                        order=order, threads=threads)
        t = oracle.time_kernel(fn, epochs=3, warmup_iters=1, min_epoch_iters=5,
                               min_epoch_time=0.1)
        if t < best:
            best, best_var = t, order
        if time.perf_counter() - t_start > budget_s:
            break
    return best, best_var


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    csr, da, x = c2_host()
    threads = len(os.sched_getaffinity(0))
    traffic = traffic_of(da.nrows, da.nnz, 4, 2, 8)
    t1, var = cpu_measure("da", da, x, threads)
    # K timed steps of a bounded sample (whole steps of 100 SpMVs when the
    # host is fast enough, else fewer SpMVs per step; the metric is a rate)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    per_step = max(1, min(SPMV_PER_STEP, int(2.0 / max(t1, 1e-9))))
    y = np.empty(da.nrows)
    for _ in range(args.warmup):
        oracle.spmv_kernel("da", da.rowptr, da.colids, da.values, x, y, 1.0, 0.0,
                           order=var, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(per_step):
            oracle.spmv_kernel("da", da.rowptr, da.colids, da.values, x, y, 1.0, 0.0,
                               order=var, threads=threads)
    el = time.perf_counter() - t0
    gbs = args.steps * per_step * traffic / el / 1e9
    sample = (f"C2 DA-CSR(i16) f64 128^3 Laplacian, {per_step} SpMVs per step, "
              f"ParallelRowBlock({threads}, '{var}') of the oracle C port; CPU {cpu_model()}")
    line = {
        "impl": "reference",
        "metric": "SpMV effective HBM GB/s (DA-CSR i16, f64)", "value": round(gbs, 3),
        "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * el / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2: 3D 7-pt Laplacian 128^3, DA-CSR i16, f64",
                   "spmv_per_step": per_step},
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
    import torch
    from paper_2307_06305_b200.harness import GraphBatch, flush_l2
    from paper_2307_06305_b200.spmv import kernel_for, resolve_variant
    kname, order = resolve_variant(variant)
    tuned = None
    if variant == "naive":
        # every exact kernel gives the same bits; run the fastest one in the
        # regime measured here (back-to-back SpMVs)
        tuned = {k: round(v * 1e6, 2) for k, v in dm.autotune(x=x, reps=20).items()}
    kname = kernel_for(dm, kname, order)
    y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dm.device)
    g = GraphBatch(lambda: dm.spmv_into(x, y, 1.0, 0.0, kname, order), per_step)
    times = gpu_steps(g, steps, warmup, flush_l2)
    # one cold SpMV at a time (L2 flushed before each) for the HBM roofline
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
    return kname, order, times, sorted(cold)[len(cold) // 2], y, tuned


def measure_e2e(a_host, x, steps, warmup, per_step):
    """Public API with pinned host buffers: x H2D and y D2H inside each call."""
    import torch
    import paper_2307_06305_b200 as dg
    xp = torch.empty(len(x), dtype=torch.float64, pin_memory=True)
    xp.numpy()[:] = x
    yp = torch.empty(a_host.nrows, dtype=torch.float64, pin_memory=True)
    xh, yh = xp.numpy(), yp.numpy()
    for _ in range(warmup):
        dg.spmv(a_host, xh, yh)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        for _ in range(per_step):
            dg.spmv(a_host, xh, yh)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    return el / steps, yh


def suite_line(name, builder):
    """GB/s of the best exact kernel on DA and CSR for one config, warm
    (graph of 20) and cold (L2 flushed before each SpMV)."""
    import torch
    from paper_2307_06305_b200.harness import time_kernel
    from paper_2307_06305_b200.spmv import kernel_for, resolve_variant
    t0 = time.time()
    mats, x, note = builder()
    out = {"build_s": round(time.time() - t0, 1), "note": note}
    for kind, dm in mats.items():
        o = dm.oindex_width // 8
        traffic = traffic_of(dm.nrows, dm.nnz, o, dm.iindex_width // 8, dm.scalar_width // 8)
        # each format runs its fastest exact kernel in each regime (all give
        # the same bits), so the DA/CSR ratio compares formats, not a policy
        # tuned for one of them
        y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dm.device)
        kname, order = resolve_variant("naive")
        dm.autotune(cold=False, x=x, reps=10)
        kwarm = kernel_for(dm, kname, order)
        fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, kwarm, order)
        warm = time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=2, min_epoch_time=0.02,
                           graph=10)
        # the layout width was chosen on the (steadier) warm timings
        dm.autotune(cold=True, x=x, tune_layout=False)
        kname = kernel_for(dm, kname, order)
        fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, kname, order)
        cold = time_kernel(fn, epochs=3, warmup_iters=1, min_epoch_iters=3, min_epoch_time=0.0,
                           cold=True)
        out[kind] = {"kernel": kname, "kernel_warm": kwarm, "bytes": traffic, "nnz": dm.nnz,
                     "warm_us": round(warm * 1e6, 2), "warm_gbs": round(traffic / warm / 1e9, 1),
                     "cold_us": round(cold * 1e6, 2), "cold_gbs": round(traffic / cold / 1e9, 1)}
        if kind == "da":
            da_choice = (kwarm, kname, dm._sliced[1].max_len if dm._sliced is not None else None,
                         dm._sliced[0].flags if dm._sliced is not None else 0)
        elif "da" in out:
            # the same kernels and slice layout as DA: the ratio then isolates
            # the format (2- vs 4-byte indices) from kernel selection
            kw, kc, t_da, flags = da_choice
            if t_da is not None:
                dm.build_slices(t_da)
                dm.set_sliced_l2_prefetch(not (flags & 1))
            fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, kw, order)
            w2 = time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=2,
                             min_epoch_time=0.02, graph=10)
            fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, kc, order)
            c2 = time_kernel(fn, epochs=3, warmup_iters=1, min_epoch_iters=3, min_epoch_time=0.0,
                             cold=True)
            out[kind]["same_kernels_as_da"] = {"warm_us": round(w2 * 1e6, 2),
                                               "cold_us": round(c2 * 1e6, 2)}
    if "da" in out and "csr" in out:
        out["uplift_cold"] = round(out["csr"]["cold_us"] / out["da"]["cold_us"], 4)
        out["uplift_predicted"] = round(out["csr"]["bytes"] / out["da"]["bytes"], 4)
        same = out["csr"].get("same_kernels_as_da")
        if same:
            out["uplift_same_kernels_warm"] = round(same["warm_us"] / out["da"]["warm_us"], 4)
            out["uplift_same_kernels_cold"] = round(same["cold_us"] / out["da"]["cold_us"], 4)
    del mats
    torch.cuda.empty_cache()
    return out


def suite_builders():
    import torch
    import paper_2307_06305_b200 as dg
    from paper_2307_06305_b200.device import DeviceMatrix
    from paper_2307_06305_b200.gen import banded_device, normal_vector
    from paper_2307_06305_b200.workloads import (laplacian_2d, laplacian_3d, skewed_rcm_laplacian,
                                                 uniform_x)
    dev = torch.device("cuda")

    def host_pair(csr, x, note):
        return ({"da": DeviceMatrix.from_host(dg.to_dacsr(csr, 16)),
                 "csr": DeviceMatrix.from_host(csr)},
                torch.from_numpy(x).to(dev), note)

    def c1():
        csr = laplacian_2d(1024)
        return host_pair(csr, uniform_x(csr.ncols, 1), "2D 5-pt 1024^2 f64 (73 MB DA: L2-resident warm)")

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

    def c3():
        m = banded_device("c3", dev)
        return m, normal_vector(m["da"].ncols, 17, dev), "random banded n=2^24 b=32767 Poisson(16)"

    def c4():
        a, info = skewed_rcm_laplacian(2048)
        return host_pair(a, uniform_x(a.ncols, 1),
                         f"2048^2 Laplacian scrambled->RCM (w {info['bandwidth_scrambled']}->"
                         f"{info['bandwidth_rcm']}) + Pareto(1.5) skew rows, max row "
                         f"{int(np.diff(a.rowptr).max())}")

    return {"c1": c1, "c2f32": c2f32, "c2bf16": c2bf16, "c3": c3, "c4": c4}


def run_c5(args, world, rank, local):
    """Config C5: 50 normalised power iterations x <- A x / ||A x|| on the
    2^28-row random banded matrix (b = 32767, Poisson(8) clamped [1, 32]),
    DA-CSR i16 with int64 rowptr, generated on the device.  One step = the
    50 iterations (50 SpMVs + 50 deterministic norms)."""
    import torch
    from paper_2307_06305_b200.device import DeviceMatrix
    from paper_2307_06305_b200.gen import banded_arrays, normal_vector
    from paper_2307_06305_b200.harness import ClockSampler
    from paper_2307_06305_b200.power import power_iteration
    from paper_2307_06305_b200.workloads import BANDED_CONFIGS
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n, b, lam, kmax, seed = BANDED_CONFIGS["c5"]
    t0 = time.time()
    arr = banded_arrays(n, b, lam, kmax, seed, dev, kinds=("da",))
    dm = DeviceMatrix("da", n, n, arr["rowptr"], arr["offsets"], arr["values"])
    x0 = normal_vector(n, 21, dev)
    build_s = time.time() - t0
    o = dm.oindex_width // 8
    traffic = traffic_of(n, dm.nnz, o, 2, 8)
    iters = 50
    # the fastest exact kernel on this operator (all give the same bits)
    tuned = {k: round(v * 1e3, 3) for k, v in
             dm.autotune(x=x0, reps=3, candidates=("sliced", "sliced_pipe", "wstream", "rowblock",
                                                   "scalar")).items()}
    kname = dm.tuned_kernel
    for _ in range(args.warmup):
        power_iteration(dm, x0, iters=2, variant=kname)
    torch.cuda.synchronize()
    times = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            _, norms = power_iteration(dm, x0, iters=iters, variant=kname)
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    step = sum(times) / len(times)
    peak, peak_src = peaks()
    line = {
        "metric": "SpMV effective HBM GB/s (DA-CSR i16, f64)",
        "value": round(iters * traffic / step / 1e9, 1), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "C5: power iteration, 50 iters, banded n=2^28 b=32767 "
                               "Poisson(8) in [1,32], DA-CSR i16 + int64 rowptr",
                   "nnz": dm.nnz, "bytes_per_spmv": traffic, "build_s": round(build_s, 1),
                   "final_norm": norms[-1], "kernel": kname,
                   "kernel_selection": "fastest exact kernel, warm ms per SpMV: "
                                       + json.dumps(tuned)},
        "roofline": {"bound": "hbm", "achieved": round(iters * traffic / step / 1e9, 1),
                     "peak": peak, "unit": "GB/s",
                     "frac": round(iters * traffic / step / 1e9 / peak, 4), "traffic": None,
                     "peak_source": peak_src},
        "gpu_launches": args.steps * iters * 3,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import paper_2307_06305_b200 as dg
    from paper_2307_06305_b200.device import DeviceMatrix
    from paper_2307_06305_b200.harness import ClockSampler

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload == "c5" and world == 1:
        return run_c5(args, world, rank, local)
    if world > 1 or args.distributed:
        from paper_2307_06305_b200 import distributed
        return distributed.bench_main(args, rank, world, local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    csr, da, xh = c2_host()
    n, nnz = da.nrows, da.nnz
    t_da = traffic_of(n, nnz, 4, 2, 8)
    t_csr = traffic_of(n, nnz, 4, 4, 8)
    dm = DeviceMatrix.of(da, dev)
    dmc = DeviceMatrix.of(csr, dev)
    x = torch.from_numpy(xh).to(dev)

    with ClockSampler(local) as clocks:
        kname, order, times, cold_da, y, tuned = measure_device(dm, x, args.variant, args.steps,
                                                                args.warmup)
    step_s = sum(times) / len(times)
    value = SPMV_PER_STEP * t_da * len(times) / sum(times) / 1e9
    # parity spot check of the benchmarked result (rows sampled vs oracle)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    yref = oracle.spmv("da", da.rowptr, da.colids, da.values, xh, threads=8)
    parity = bool(np.array_equal(y.cpu().numpy().view(np.uint64), yref.view(np.uint64)))

    kc, _, times_c, cold_csr, _, _ = measure_device(dmc, x, args.variant,
                                                    max(3, args.steps // 2), 2)
    step_c = sum(times_c) / len(times_c)

    e2e_step, _ = measure_e2e(da, xh, max(2, args.steps // 5), 1, SPMV_PER_STEP // 10)
    e2e_spmv = SPMV_PER_STEP // 10
    e2e_gbs = e2e_spmv * t_da / e2e_step / 1e9

    peak, peak_src = peaks()
    per_launch = step_s / SPMV_PER_STEP
    achieved = t_da / per_launch / 1e9
    traffic, steady = ncu_traffic(kname + ":c2:da")
    steady_bytes = steady.get("dram_bytes_per_launch") if steady else None
    line = {
        "metric": "SpMV effective HBM GB/s (DA-CSR i16, f64)",
        "value": round(value, 1), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2: 3D 7-pt Laplacian 128^3 (n=2097152, nnz=14581760), DA-CSR "
                               "i16 offsets, f64, x~U[-1,1] seed 1",
                   "spmv_per_step": SPMV_PER_STEP, "kernel": kname,
                   "kernel_selection": "fastest exact kernel (bit-identical results), warm "
                                       "autotune in us per SpMV: " + json.dumps(tuned),
                   "l2": "188 MB matrix > 126 MB L2; L2 flushed (read of 2x L2, clean lines) before every step",
                   "parallelism": "1 GPU"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_source": "ncu --set full, one cold launch (profiles/)",
                     "traffic_steady_state": steady_bytes,
                     "traffic_steady_state_note": steady.get("note") if steady else None,
                     "dram_gbs_steady_state": (round(steady_bytes / per_launch / 1e9, 1)
                                               if steady_bytes else None),
                     "dram_frac_steady_state": (round(steady_bytes / per_launch / 1e9 / peak, 4)
                                                if steady_bytes else None),
                     "peak_source": peak_src, "bytes_per_launch": t_da,
                     "frac_of_nominal_8TBs": round(achieved / 8000.0, 4),
                     "frac_of_tma_read_ceiling": round(achieved / READ_CEILING_GBS, 4),
                     "read_ceiling_note": f"{READ_CEILING_GBS} GB/s = pure TMA bulk-copy "
                                          "read stream measured by tools/peaks.py (SpMV is "
                                          "~91% reads; the copy peak counts writes too)",
                     "cold_single_spmv_gbs": round(t_da / cold_da / 1e9, 1)},
        "csr_comparator": {"kernel": kc, "value": round(SPMV_PER_STEP * t_csr / step_c / 1e9, 1),
                           "unit": "GB/s", "bytes_per_spmv": t_csr,
                           "uplift_measured": round(step_c / step_s, 4),
                           "uplift_measured_cold_single": round(cold_csr / cold_da, 4),
                           "uplift_predicted": round(t_csr / t_da, 4)},
        "e2e": {"value": round(e2e_gbs, 1), "unit": "GB/s",
                "h2d_bytes_per_step": e2e_spmv * n * 8, "d2h_bytes_per_step": e2e_spmv * n * 8,
                "spmv_per_step": e2e_spmv,
                "note": "spmv(A, x_host, y_host) public API, pinned host x/y; operator resident"},
        "gflops": round(SPMV_PER_STEP * dg.work_flops(nnz=nnz, nrows=n) / step_s / 1e9, 1),
        "parity_bit_exact_vs_oracle": parity,
        "gpu_launches": args.steps * SPMV_PER_STEP,
        "clocks": clocks.summary(),
    }
    if not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        t_cpu, var = cpu_measure("da", da, xh, threads)
        # thread scaling of the same CPU path (T = 1, 2, 4, 8, all)
        import oracle
        y_cpu = np.empty(da.nrows)
        scaling = {}
        for t in sorted({1, 2, 4, 8, threads}):
            if t > threads:
                continue
            fn = lambda t=t: oracle.spmv_kernel("da", da.rowptr, da.colids, da.values, xh, y_cpu,
                                                1.0, 0.0, order=var, threads=t)
            tt = oracle.time_kernel(fn, epochs=2, warmup_iters=1, min_epoch_iters=2,
                                    min_epoch_time=0.05)
            scaling[str(t)] = round(t_da / tt / 1e9, 2)
        line["cpu_baseline"] = {
            "value": round(t_da / t_cpu / 1e9, 3), "unit": "GB/s", "cores": threads,
            "gbs_by_threads": scaling,
            "kind": "port",
            "sample": f"C2 DA-CSR f64, one SpMV per iteration, best of the reference inner "
                      f"variants ('{var}' won) under ParallelRowBlock({threads}), 3 epochs of "
                      f">=5 iters/>=0.1 s; oracle C port of _numba_kernels; CPU {cpu_model()}"}
    if not args.no_suite:
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
