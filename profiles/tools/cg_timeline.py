"""Dev tool: CUPTI timeline of 2 device-resident CG iterations at configs[1]
(btg_cg_solve), per kernel, to compare one iteration with one Hessian."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2407_13066_b200 as btg  # noqa: E402

cfg = bench.CONFIGS["B"]
op = bench.build_operator(cfg, 0, seed=1000)
m = torch.empty((cfg["nm"], cfg["nt"]), dtype=torch.float64, device="cuda:0")
btg.fill_uniform(m, seed=7)
if os.environ.get("HOST_FIRST"):  # host-buffer calls first (the bench's e2e leg)
    from paper_2407_13066_b200 import _lib

    hm = torch.empty((cfg["nm"], cfg["nt"]), dtype=torch.float64, pin_memory=True)
    hm.copy_(m.cpu())
    out_d = torch.empty((cfg["nd"], cfg["nt"]), dtype=torch.float64, pin_memory=True).numpy()
    L = _lib.load()
    op._bind_stream(None)
    for _ in range(3):
        _lib.check(L.btg_forward(op._h, hm.numpy().ctypes.data, hm.numel(), out_d.ctypes.data, out_d.size, 1, 0))
btg.cg_solve_op(op, m, alpha=1e-2, tol=0.0, maxiter=1)
torch.cuda.synchronize()
for iters in (1, 2, 5):
    t = time.perf_counter()
    btg.cg_solve_op(op, m, alpha=1e-2, tol=0.0, maxiter=iters)
    torch.cuda.synchronize()
    print(f"cg {iters} iterations: {(time.perf_counter() - t) * 1e3:.2f} ms wall")
t = time.perf_counter()
for _ in range(5):
    op.hessian_apply(m, alpha=1e-2)
torch.cuda.synchronize()
print(f"hessian x5: {(time.perf_counter() - t) * 1e3:.2f} ms wall")
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    btg.cg_solve_op(op, m, alpha=1e-2, tol=0.0, maxiter=2)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in evs)
for e in sorted(evs, key=lambda e: e.time_range.start):
    print(f"  {(e.time_range.start - t0) / 1e3:8.3f} +{(e.time_range.end - e.time_range.start) / 1e3:7.3f} ms"
          f"  ch{getattr(e, 'device_resource_id', '?')}  {e.name[:60]}")
