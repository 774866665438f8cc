"""Measure the read-stream ceilings on this B200 (for the roofline notes):
torch copy (same method as MEASURED_PEAKS.json), torch sum (read-only),
and the library's TMA bulk-copy stream probe over chunk sizes / CTA counts."""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2307_06305_b200 import _native

dev = torch.device("cuda")
nbytes = 4 << 30
buf = torch.ones(nbytes // 8, dtype=torch.float64, device=dev)
out = torch.empty_like(buf[: nbytes // 16])


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


res = {}
half = buf[: nbytes // 16]
res["torch_copy_gbs(read+write)"] = 2 * half.numel() * 8 / timed(lambda: out.copy_(half)) / 1e9
res["torch_sum_gbs(read)"] = nbytes / timed(lambda: buf.sum()) / 1e9
sink = torch.zeros(1, dtype=torch.float64, device=dev)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
L = _native.lib()
for chunk in (2048, 4096, 8192, 12288):
    for per_sm in (2, 3, 4, 6):
        ctas = sms * per_sm
        if chunk * 16 * per_sm > 220 * 1024:
            continue
        def run():
            _native.check(L.dacsr_stream_probe(ctypes.c_void_p(buf.data_ptr()), nbytes, chunk, ctas,
                                               ctypes.c_void_p(sink.data_ptr()),
                                               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
                          "probe")
        res[f"tma_probe_chunk{chunk}_ctas{per_sm}x"] = nbytes / timed(run) / 1e9
print(json.dumps({k: round(v, 1) for k, v in res.items()}, indent=1))
