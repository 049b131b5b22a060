"""compute-sanitizer workload for the session-4 kernels (dev tool): the transposed
setup (k_tosi_to_soti + vector R2C, FP64 and the FP32 rounding kernel
k_spec_to_f32), the light C2R instantiations (k_c2r_tma / k_c2r_pf / k_c2r_fast
with <..., LIGHT = true>), the re-strided N_t = 1000 / 4096 plans, and the TMA
ZGEMM adjoint with one 4-D box per operand and stage plus its constant-offset
epilogue (N_d a multiple of 8). Run plainly it prints the max rel L2 against the
oracle (1.3e-15, round 2 session 4); compute-sanitizer is closed on the GPU pool
for this round, so the tool runs of `r02s2_sanitizer.md` could not be repeated."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch  # noqa: E402

import paper_2407_13066_b200 as btg  # noqa: E402
from oracle import restate as R  # noqa: E402

errs = []
rng = np.random.default_rng(4)
# multi-RHS, N_t = 1024: blocked TMA R2C, light / full k_c2r_tma, chunked TMA adjoint
nt, nd, nm, nrhs = 1024, 24, 136, 5
blocks, _, _ = R.random_problem(79, nd, nm, nt)
spec = R.setup_full(blocks)
M = rng.uniform(-1, 1, size=(nrhs, nm, nt))
D = rng.uniform(-1, 1, size=(nrhs, nd, nt))
with btg.setup(torch.from_numpy(blocks).cuda()) as op:
    Md, Dd = torch.from_numpy(M).cuda(), torch.from_numpy(D).cuda()
    F = op.apply_forward(Md).cpu().numpy()
    A = op.apply_adjoint(Dd).cpu().numpy()
    H = op.hessian_apply(Md, alpha=0.1, reg="temporal-laplacian").cpu().numpy()
    errs += [R.rel_l2(F[r], R.apply_forward(spec, M[r])) for r in range(nrhs)]
    errs += [R.rel_l2(A[r], R.apply_adjoint(spec, D[r])) for r in range(nrhs)]
    errs.append(R.rel_l2(H[1], R.gauss_newton_apply(spec, M[1], None, 0.1, 1)))
    # single RHS: frequency-major light k_c2r_pf
    errs.append(R.rel_l2(op.apply_adjoint(D[0]), R.apply_adjoint(spec, D[0])))
# N_t = 1000 / 4096 (light k_c2r_fast, new channel strides), FP64 and FP32 F-hat setup
for nt2, nd2, nm2 in ((1000, 3, 40), (4096, 2, 17)):
    b2, m2, d2 = R.random_problem(nt2 + 1, nd2, nm2, nt2)
    s2 = R.setup_full(b2)
    with btg.setup(b2) as op:
        errs.append(R.rel_l2(op.apply_forward(m2), R.apply_forward(s2, m2)))
        errs.append(R.rel_l2(op.apply_adjoint(d2), R.apply_adjoint(s2, d2)))
    with btg.setup(b2, precision=32) as op:
        assert R.rel_l2(op.spectrum(), s2[: nt2 + 1]) <= 1e-7
print("max rel L2", max(errs))
