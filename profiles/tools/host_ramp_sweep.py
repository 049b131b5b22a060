"""Dev tool: end-to-end (host-buffer) F / F* / H times at configs[1] for one
setting of the host-pipeline knobs (BTG_HOST_RAMP etc. read from the env).
Usage on the GPU box: BTG_HOST_RAMP=150 python profiles/tools/host_ramp_sweep.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_13066_b200 as btg  # noqa: E402
from paper_2407_13066_b200 import _lib  # noqa: E402

cfg = dict(bench.CONFIGS[os.environ.get("CFG", "B")], precision=int(os.environ.get("PREC", "64")))
nt, nd, nm = cfg["nt"], cfg["nd"], cfg["nm"]
op = bench.build_operator(cfg, 0, seed=1000)
m = torch.empty((nm, nt), dtype=torch.float64, device="cuda:0")
btg.fill_uniform(m, seed=7)
hm = torch.empty((nm, nt), dtype=torch.float64, pin_memory=True)
hm.copy_(m.cpu())
hd = torch.empty((nd, nt), dtype=torch.float64, pin_memory=True).normal_()
hg = torch.linspace(0.5, 2.0, nd, dtype=torch.float64).numpy()
hm_np, hd_np = hm.numpy(), hd.numpy()
out_d = torch.empty((nd, nt), dtype=torch.float64, pin_memory=True).numpy()
out_m = torch.empty((nm, nt), dtype=torch.float64, pin_memory=True).numpy()
L = _lib.load()
op._bind_stream(None)
ts = {"F": [], "F*": [], "H": []}
for it in range(12):
    t0 = time.perf_counter()
    _lib.check(L.btg_forward(op._h, hm_np.ctypes.data, hm_np.size, out_d.ctypes.data, out_d.size, 1, 0))
    t1 = time.perf_counter()
    _lib.check(L.btg_adjoint(op._h, hd_np.ctypes.data, hd_np.size, out_m.ctypes.data, out_m.size, 1, 0))
    t2 = time.perf_counter()
    _lib.check(L.btg_hessian(op._h, hm_np.ctypes.data, hm_np.size, out_m.ctypes.data, out_m.size, 1,
                             hg.ctypes.data, 1, 0.0, 0, 0))
    t3 = time.perf_counter()
    if it >= 2:
        for k, dt in zip(ts, (t1 - t0, t2 - t1, t3 - t2)):
            ts[k].append(dt * 1e3)
tag = " ".join(f"{k}={os.environ[k]}" for k in sorted(os.environ) if k.startswith("BTG_"))
print(f"{tag or 'default'}: " + " ".join(f"{k} {statistics.median(v):.3f}" for k, v in ts.items())
      + f" sum {sum(statistics.median(v) for v in ts.values()):.3f} ms")
