"""compute-sanitizer workload for the round-2 kernels (dev tool): the
warp-specialised TMA 3M ZGEMM with the channel-blocked spectrum (N_t = 1024:
blocked TMA R2C, k_c2r_tma), the device-pointer Hessian graph replay, the CG
graph (WHILE node, folded p^T H p) and the P2P grid with the reduce fused into
the C2R."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch  # noqa: E402

import paper_2407_13066_b200 as btg  # noqa: E402
from oracle import restate as R  # noqa: E402
from paper_2407_13066_b200.distributed import Partition  # noqa: E402

nt, nd, nm, nrhs = 1024, 20, 136, 5
blocks, _, _ = R.random_problem(78, nd, nm, nt)
spec = R.setup_full(blocks)
rng = np.random.default_rng(2)
M = rng.uniform(-1, 1, size=(nrhs, nm, nt))
D = rng.uniform(-1, 1, size=(nrhs, nd, nt))
errs = []
with btg.setup(blocks) as op:
    Md, Dd = torch.from_numpy(M).cuda(), torch.from_numpy(D).cuda()
    F = op.apply_forward(Md).cpu().numpy()
    A = op.apply_adjoint(Dd).cpu().numpy()
    for _ in range(2):  # second call replays the captured Hessian graph
        H = op.hessian_apply(Md, alpha=0.1, reg="temporal-laplacian").cpu().numpy()
    errs += [R.rel_l2(F[r], R.apply_forward(spec, M[r])) for r in range(nrhs)]
    errs += [R.rel_l2(A[r], R.apply_adjoint(spec, D[r])) for r in range(nrhs)]
    errs.append(R.rel_l2(H[1], R.gauss_newton_apply(spec, M[1], None, 0.1, 1)))
    x, it, res, conv = btg.cg_solve_op(op, torch.from_numpy(R.apply_adjoint(spec, D[0])).cuda(), alpha=0.05,
                                       tol=1e-9, maxiter=50)
with Partition(blocks[:256].copy(), (2, 3)) as p:
    f = p.forward(M[0][:, :256].copy())
    errs.append(R.rel_l2(f, R.apply_forward(R.setup_full(blocks[:256].copy()), M[0][:, :256].copy())))
print("max rel L2", max(errs), "cg iterations", it, "residual", res)
