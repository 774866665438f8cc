"""ncu driver: config C3 (random banded n=2^24, b=32767), one kernel."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2307_06305_b200.gen import banded_device, normal_vector
from paper_2307_06305_b200.harness import flush_l2
from paper_2307_06305_b200.spmv import kernel_for, resolve_variant

m = banded_device("c3", "cuda", kinds=("da",))["da"]
x = normal_vector(m.ncols, 17, "cuda")
y = torch.empty(m.nrows, dtype=torch.float64, device="cuda")
for v in (sys.argv[1] if len(sys.argv) > 1 else "naive").split(","):
    k, o = resolve_variant(v)
    k = kernel_for(m, k, o)
    for _ in range(2):
        flush_l2()
        m.spmv_into(x, y, 1.0, 0.0, k, o)
torch.cuda.synchronize()
print("ok")
