"""GPU timing harness in the reference's methodology.

``time_kernel`` follows /root/reference/pkg/src/dacsr/bench.py:96-115
(warm-up, then epochs that each repeat until both a minimum iteration count
and a minimum time are met; the result is the minimum per-iteration time)
but times on the device with CUDA events on the launching stream, with a
synchronize on both sides.  ``flush_l2`` writes a buffer twice the size of
the L2 so a measurement can start cold.
"""

import math
import subprocess
import threading
import time

import torch

_flush_buf = {}


def l2_bytes(device=None):
    props = torch.cuda.get_device_properties(device or torch.cuda.current_device())
    return int(getattr(props, "L2_cache_size", 126 << 20) or (126 << 20))


def flush_l2(device=None, stream=None):
    """Evict L2 by READING 2x L2 worth of memory.

    A write-based flush leaves L2 full of dirty lines whose write-back then
    lands inside the next timed region; reading leaves clean lines, so the
    measured kernel pays only for its own traffic."""
    device = torch.device(device or "cuda")
    buf = _flush_buf.get(device)
    if buf is None:
        buf = torch.ones(2 * l2_bytes(device) // 4, dtype=torch.int32, device=device)
        _flush_buf[device] = (buf, torch.empty((), dtype=torch.int64, device=device))
    buf, out = _flush_buf[device]
    with torch.cuda.stream(stream or torch.cuda.current_stream(device)):
        torch.sum(buf, 0, out=out)


class GraphBatch:
    """``n`` back-to-back calls of ``fn`` captured once in a CUDA graph, so
    replays carry no host launch overhead between kernels."""

    def __init__(self, fn, n, stream=None):
        self.n = n
        fn()  # warm: lazy init, launch-config caches
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        s = stream or torch.cuda.Stream()
        with torch.cuda.graph(self.graph, stream=s):
            for _ in range(n):
                fn()
        torch.cuda.synchronize()

    def __call__(self):
        self.graph.replay()


def time_kernel(fn, epochs=11, warmup_iters=10, min_epoch_iters=10, min_epoch_time=0.1,
                stream=None, cold=False, graph=0):
    """Best-of-epochs per-iteration seconds of ``fn`` measured with CUDA events.

    With ``cold=True`` every iteration is timed individually after an L2
    flush (the flush is outside the events) and the epoch time is the sum of
    the per-iteration event times.  With ``graph=n`` (warm mode) ``fn`` is
    captured n times into a CUDA graph that is replayed instead.
    """
    stream = stream or torch.cuda.current_stream()
    per_call = 1
    if graph and not cold:
        fn = GraphBatch(fn, graph)
        per_call = graph
    for _ in range(warmup_iters):
        fn()
    torch.cuda.synchronize()
    best = math.inf
    for _ in range(epochs):
        iters, elapsed = 0, 0.0
        if cold:
            while iters < min_epoch_iters or elapsed < min_epoch_time:
                flush_l2(stream=stream)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                e1.synchronize()
                elapsed += e0.elapsed_time(e1) / 1e3
                iters += 1
        else:
            # the epoch repeats fn until both min_epoch_iters and
            # min_epoch_time of DEVICE time are covered; the count comes from
            # the device time of one batch (a host-time loop would enqueue far
            # more work than intended when one call is milliseconds long)
            batch = max(1, min_epoch_iters)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(batch):
                fn()
            e1.record(stream)
            e1.synchronize()
            t_batch = max(e0.elapsed_time(e1) / 1e3, 1e-9)
            reps = max(1, min(1_000_000 // batch, math.ceil(min_epoch_time / t_batch)))
            e0.record(stream)
            for _ in range(reps * batch):
                fn()
            e1.record(stream)
            e1.synchronize()
            iters = reps * batch
            elapsed = e0.elapsed_time(e1) / 1e3
        best = min(best, elapsed / (iters * per_call))
    return best


class ClockSampler:
    """Samples nvidia-smi clocks / throttle reasons while running."""

    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, period_ms=20):
        self.index = index
        self.period_ms = period_ms
        self.rows = []
        self._proc = None
        self._thread = None

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", f"-lms={self.period_ms}"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._thread = threading.Thread(target=self._read, daemon=True)
            self._thread.start()
        except OSError:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()
            self._thread.join(timeout=5)
            if not self.rows:  # region shorter than the period: one sample at its end
                try:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=10).stdout
                    for line in out.splitlines():
                        parts = [p.strip() for p in line.split(",")]
                        if len(parts) >= 8:
                            self.rows.append(parts)
                except (OSError, subprocess.TimeoutExpired):
                    pass

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if not self.rows:
            why = "nvidia-smi unavailable" if self._proc is None else \
                "no sample: timed region shorter than the sampling period"
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [why], "samples": 0}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[4 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}
