"""ncu driver: a few SpMVs of config C4 (skewed, RCM-ordered) with one kernel."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import flush_l2
from paper_2307_06305_b200.spmv import kernel_for, resolve_variant
from paper_2307_06305_b200.workloads import skewed_rcm_laplacian, uniform_x

a, info = skewed_rcm_laplacian(2048)
dm = DeviceMatrix.from_host(dg.to_dacsr(a, 16))
x = torch.from_numpy(uniform_x(a.ncols, 1)).cuda()
y = torch.empty(a.nrows, dtype=torch.float64, device="cuda")
for v in (sys.argv[1] if len(sys.argv) > 1 else "naive").split(","):
    k, o = resolve_variant(v)
    k = kernel_for(dm, k, o)
    for _ in range(2):
        flush_l2()
        dm.spmv_into(x, y, 1.0, 0.0, k, o)
torch.cuda.synchronize()
print("ok")
