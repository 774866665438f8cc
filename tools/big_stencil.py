import sys, json, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2307_06305_b200 as dg
from paper_2307_06305_b200.device import DeviceMatrix
from paper_2307_06305_b200.harness import time_kernel
from paper_2307_06305_b200.model import StorageWidths, spmv_traffic
from paper_2307_06305_b200.workloads import laplacian_3d, laplacian_3d_box, uniform_x
dev = torch.device("cuda")
for g, dt in ((128, np.float64), ((1024, 128, 128), np.float64), ((1024, 128, 128), np.float32),
              (256, np.float64)):
    t0 = time.time()
    csr = laplacian_3d(g, dt) if isinstance(g, int) else laplacian_3d_box(g, dt)
    da = dg.to_dacsr(csr, 32 if isinstance(g, int) and g * g > 32767 else 16)
    mats = {"csr": DeviceMatrix.from_host(csr), "da": DeviceMatrix.from_host(da)}
    x = torch.from_numpy(uniform_x(csr.ncols, 1).astype(dt)).to(dev)
    for kind, dm in mats.items():
        tr = spmv_traffic(dm.nrows, dm.ncols, dm.nnz, StorageWidths(dm.oindex_width // 8, dm.iindex_width // 8, dm.scalar_width // 8)).total_bytes
        y = torch.empty(dm.nrows, dtype=dm.values.dtype, device=dev)
        fn = lambda: dm.spmv_into(x, y, 1.0, 0.0, "sliced_pipe", 0)
        warm = time_kernel(fn, epochs=3, warmup_iters=2, min_epoch_iters=3, min_epoch_time=0.0, graph=10)
        cold = time_kernel(fn, epochs=3, warmup_iters=1, min_epoch_iters=4, min_epoch_time=0.0, cold=True)
        print(json.dumps({"grid": g, "dtype": str(np.dtype(dt)), "kind": kind, "inner_bits": dm.iindex_width, "bytes": tr, "warm_us": round(warm*1e6,1), "cold_us": round(cold*1e6,1), "warm_gbs": round(tr/warm/1e9), "cold_gbs": round(tr/cold/1e9)}), flush=True)
    print("host build + upload s", round(time.time() - t0, 1), flush=True)
    del mats
    torch.cuda.empty_cache()
