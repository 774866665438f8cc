"""Small driver for compute-sanitizer (memcheck / racecheck): every kernel
variant on a few golden-corpus matrices incl. empty rows, rectangular and
long-row cases, f32/f64, DA/CSR, plus the plan / conversion / norm kernels."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "oracle")
import numpy as np
import torch

import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix, bandwidth_device, to_dacsr_device
from paper_2307_06305_b200.power import chunked_sumsq
from test_oracle import CORPUS

dev = torch.device("cuda")
picked = [c for c in CORPUS if c["nrows"] and c["ncols"]][:12] + [CORPUS[1]]
bad = 0
for c in picked:
    for kind, inner in (("csr", "colids"), ("da", "offsets")):
        cls = dg.CsrMatrix if kind == "csr" else dg.DacsrMatrix
        a = cls(c["nrows"], c["ncols"], c["rowptr"], c[inner], c["values"])
        dm = DeviceMatrix.from_host(a, dev)
        x = torch.from_numpy(c["x"]).to(dev)
        for v in ("wstream", "rowblock", "staged", "scalar", "vector4", "warp", "rowblock_tree",
                  "multi_accumulator_3", "strip_mined_4"):
            y = torch.from_numpy(c["y0"].copy()).to(dev)
            dg.spmv(dm, x, y, c["alpha"] or 1.0, c["beta"], v)
            want = c["y_naive"] if c["alpha"] else None
        if kind == "csr":
            bandwidth_device(dm)
            if dg.bandwidth(a) < 32767:
                to_dacsr_device(dm, 16)
    chunked_sumsq(torch.from_numpy(c["x"]).to(dev), 64)
torch.cuda.synchronize()
print("sanitize driver done")
