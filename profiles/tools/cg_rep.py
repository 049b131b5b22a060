import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch, bench
import paper_2407_13066_b200 as btg
from paper_2407_13066_b200 import _lib
cfg = bench.CONFIGS["B"]; nt, nd, nm = cfg["nt"], cfg["nd"], cfg["nm"]
op = bench.build_operator(cfg, 0, seed=1000)
m = torch.empty((nm, nt), dtype=torch.float64, device="cuda:0"); btg.fill_uniform(m, seed=7)
stream = torch.cuda.current_stream(0)
def cg_time(tag):
    btg.cg_solve_op(op, m, alpha=1e-2, tol=0.0, maxiter=1)
    torch.cuda.synchronize()
    c0 = torch.cuda.Event(enable_timing=True); c1 = torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    c0.record(stream)
    _, it, _, _ = btg.cg_solve_op(op, m, alpha=1e-2, tol=0.0, maxiter=20)
    c1.record(stream)
    torch.cuda.synchronize()
    print(tag, it, c0.elapsed_time(c1) / it, (time.perf_counter() - t) * 1e3 / it)
cg_time("fresh")
hm = torch.empty((nm, nt), dtype=torch.float64, pin_memory=True); hm.copy_(m.cpu())
out_d = torch.empty((nd, nt), dtype=torch.float64, pin_memory=True).numpy()
L = _lib.load(); op._bind_stream(None)
hm_np = hm.numpy()
for _ in range(3):
    _lib.check(L.btg_forward(op._h, hm_np.ctypes.data, hm_np.size, out_d.ctypes.data, out_d.size, 1, 0))
cg_time("after host calls")
