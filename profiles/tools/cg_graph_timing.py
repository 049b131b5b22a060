"""CG ms/iteration, graph loop (default) vs host loop (BTG_CG_HOST_LOOP=1), at
configs[0] (launch-bound) and an N_m slice of configs[1]. Dev tool only."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np, torch
import paper_2407_13066_b200 as btg
from oracle import restate as R

def run(blocks, iters, reps=5):
    out = {}
    with btg.setup(blocks) as op:
        nm, nt = blocks.shape[2], blocks.shape[0]
        m = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (nm, nt))).cuda()
        for mode in ("graph", "host"):
            if mode == "host":
                os.environ["BTG_CG_HOST_LOOP"] = "1"
            else:
                os.environ.pop("BTG_CG_HOST_LOOP", None)
            btg.cg_solve_op(op, m, alpha=1e-2, tol=0.0, maxiter=iters)
            torch.cuda.synchronize()
            best = 1e30
            for _ in range(reps):
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(); _, it, _, _ = btg.cg_solve_op(op, m, alpha=1e-2, tol=0.0, maxiter=iters); e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / it)
            out[mode] = best
        os.environ.pop("BTG_CG_HOST_LOOP", None)
    return out

res = {}
b0, _, _ = R.random_problem(1, 8, 256, 64)
res["configs[0] N_t=64 N_d=8 N_m=256 (200 it)"] = run(b0, 200)
rng = np.random.default_rng(5)
b1 = rng.uniform(-1, 1, (1024, 100, 2048))
res["configs[1] slice N_t=1024 N_d=100 N_m=2048 (20 it)"] = run(b1, 20)
print(json.dumps(res, indent=1))

# device-pointer Hessian call: graph replay (default) vs eager chain (BTG_NO_GRAPH=1)
from paper_2407_13066_b200 import _lib
L = _lib.load()
hres = {}
for name, blocks in (("configs[0]", b0), ("configs[1] slice N_m=2048", b1)):
    with btg.setup(blocks) as op:
        nt, nd, nm = blocks.shape
        v = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, (nm, nt))).cuda()
        out = torch.empty_like(v)
        op._bind_stream(v)
        for mode in ("graph", "eager"):
            if mode == "eager":
                os.environ["BTG_NO_GRAPH"] = "1"
            else:
                os.environ.pop("BTG_NO_GRAPH", None)
            call = lambda: _lib.check(L.btg_hessian(op._h, v.data_ptr(), v.numel(), out.data_ptr(), out.numel(), 1,
                                                    None, 0, 0.1, 1, _lib.BTG_DEVICE_PTRS))
            for _ in range(5):
                call()
            torch.cuda.synchronize()
            n = 200 if name == "configs[0]" else 20
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                call()
            e1.record(); torch.cuda.synchronize()
            hres[f"{name} {mode}"] = e0.elapsed_time(e1) / n
        os.environ.pop("BTG_NO_GRAPH", None)
print(json.dumps({"hessian_ms_per_call": hres}, indent=1))
