"""Timeline of the streamed host pipeline (C2, 4 pieces), rebuilt with torch
copies + timing events, to see where the e2e call loses time against the
PCIe model."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200 import hostpath
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.workloads import laplacian_3d, uniform_x

csr = laplacian_3d(128)
da = dg.to_dacsr(csr, 16)
n = csr.nrows
x = uniform_x(n, 1)
xp = torch.empty(n, dtype=torch.float64, pin_memory=True); xp.numpy()[:] = x
yp = torch.empty(n, dtype=torch.float64, pin_memory=True)
dm = DeviceMatrix.of(da)
sh = hostpath.StreamedHost(dm, 4)
xd, yd = sh.x, sh.y
h2d, comp, d2h = sh.s_h2d, sh.s_comp, sh.s_d2h
w = sh.w
P = len(sh.views)


def ev(s):
    e = torch.cuda.Event(enable_timing=True)
    e.record(s)
    return e


def one(copy_only=False, serial=False):
    t = {}
    start = ev(torch.cuda.current_stream())
    h2d.wait_event(start); comp.wait_event(start); d2h.wait_event(start)
    sent = 0
    for p, v in enumerate(sh.views):
        r0, r1 = v.row_start, v.row_end
        hi = min(n, r1 + w)
        with torch.cuda.stream(h2d):
            if serial and p:
                h2d.wait_event(t[f"d2h{p-1}_end"])
            xd[sent:hi].copy_(xp[sent:hi], non_blocking=True)
            sent = hi
            t[f"h2d{p}_end"] = ev(h2d)
        comp.wait_event(t[f"h2d{p}_end"])
        with torch.cuda.stream(comp):
            t[f"k{p}_start"] = ev(comp)
            if not copy_only:
                v.spmv_into(xd, yd, 1.0, 0.0, "wstream", 0, stream=comp)
            t[f"k{p}_end"] = ev(comp)
        d2h.wait_event(t[f"k{p}_end"])
        with torch.cuda.stream(d2h):
            t[f"d2h{p}_start"] = ev(d2h)
            yp[r0:r1].copy_(yd[r0:r1], non_blocking=True)
            t[f"d2h{p}_end"] = ev(d2h)
    d2h.synchronize()
    return start, t


for mode in ("full", "copy_only", "serial"):
    for _ in range(3):
        one(mode == "copy_only", mode == "serial")
    start, t = one(mode == "copy_only", mode == "serial")
    torch.cuda.synchronize()
    line = {k: round(start.elapsed_time(e) * 1e3, 1) for k, e in t.items()}
    print(mode, "total us", line[f"d2h{P-1}_end"])
    print("  ", line)
