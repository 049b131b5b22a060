import sys, numpy as np
import os; sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import paper_2407_13066_b200 as btg
from oracle import restate as R
nd, nm, nt, nrhs = 20, 4500, 16, 5
blocks, _, _ = R.random_problem(77, nd, nm, nt)
spec = R.setup_full(blocks)
rng = np.random.default_rng(1)
M = rng.uniform(-1, 1, size=(nrhs, nm, nt)); D = rng.uniform(-1, 1, size=(nrhs, nd, nt))
with btg.setup(blocks) as op:
    F = op.apply_forward(M); A = op.apply_adjoint(D); H = op.hessian_apply(M, alpha=0.1)
    f1 = op.apply_forward(M[0]); a1 = op.apply_adjoint(D[0])
print(max(R.rel_l2(F[r], R.apply_forward(spec, M[r])) for r in range(nrhs)), R.rel_l2(f1, R.apply_forward(spec, M[0])))
