"""Host-pointer calls with N_m >= 4096 stream the long vector in column chunks
overlapped with the GEMV (btg_capi.cu host_forward_stage / host_adjoint_stage).
Check them against the device-pointer path and the oracle, including a ragged
last chunk, the Gamma^-1 / alpha R v epilogues and FP32 F-hat."""

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def btg():
    import paper_2407_13066_b200 as m

    return m


@pytest.mark.parametrize("nm,nt", [(4096, 64), (5000, 64), (9000, 64), (4100, 15)])
def test_chunked_host_path_matches_device_path(btg, nm, nt):
    import torch

    nd = 7
    blocks, m, d = R.random_problem(1300 + nm, nd, nm, nt)
    spec = R.setup_full(blocks)
    gam = np.linspace(0.5, 2.0, nd)
    with btg.setup(blocks) as op:
        f_host = op.apply_forward(m)
        a_host = op.apply_adjoint(d)
        h_host = op.hessian_apply(m, alpha=0.2, reg="temporal-laplacian", gamma_inv=gam)
        f_dev = op.apply_forward(torch.from_numpy(m).cuda()).cpu().numpy()
        a_dev = op.apply_adjoint(torch.from_numpy(d).cuda()).cpu().numpy()
        h_dev = op.hessian_apply(torch.from_numpy(m).cuda(), alpha=0.2, reg="temporal-laplacian",
                                 gamma_inv=torch.from_numpy(gam).cuda()).cpu().numpy()
        # epilogue-extended entry points through the host path too
        fg = op.apply_forward(m, gamma_inv=gam)
        ar = op.apply_adjoint(d, reg_v=m, alpha=0.3, reg="temporal-laplacian")
        # repeated host calls are bit-identical
        assert np.array_equal(f_host, op.apply_forward(m))
    assert R.rel_l2(f_host, R.apply_forward(spec, m)) <= 1e-12
    assert R.rel_l2(a_host, R.apply_adjoint(spec, d)) <= 1e-12
    assert R.rel_l2(h_host, R.gauss_newton_apply(spec, m, gam, 0.2, 1)) <= 1e-12
    assert R.rel_l2(f_host, f_dev) <= 1e-14
    assert np.array_equal(a_host, a_dev)  # adjoint chunks partition columns: identical arithmetic
    assert R.rel_l2(h_host, h_dev) <= 1e-14
    assert R.rel_l2(fg, gam[:, None] * R.apply_forward(spec, m)) <= 1e-12
    assert R.rel_l2(ar, R.apply_adjoint(spec, d) + 0.3 * R.reg_apply(m, 1)) <= 1e-12


def test_chunked_host_path_fp32(btg):
    blocks, m, d = R.random_problem(1400, 5, 6000, 32)
    spec = R.setup_full(blocks)
    with btg.setup(blocks, precision=32) as op:
        assert R.rel_l2(op.apply_forward(m), R.apply_forward(spec, m)) <= 1e-5
        assert R.rel_l2(op.apply_adjoint(d), R.apply_adjoint(spec, d)) <= 1e-5
        assert R.rel_l2(op.hessian_apply(m, alpha=0.1), R.hessian_apply(spec, m, 0.1, 0)) <= 1e-5


@pytest.mark.parametrize("kind", ["sensor", "sample"])
def test_chunked_adjoint_gamma_epilogue_offsets(btg, kind):
    """A Gamma-weighted adjoint output (btg_adjoint_ex, gamma over the N_m output
    channels) through the column-chunked host path: each chunk's epilogue reads
    Gamma at its own column offset."""
    nd, nm, nt = 6, 5000, 32
    blocks, _, d = R.random_problem(1500, nd, nm, nt)
    spec = R.setup_full(blocks)
    rng = np.random.default_rng(3)
    g = rng.uniform(0.5, 2.0, size=(nm,) if kind == "sensor" else (nm, nt))
    with btg.setup(blocks) as op:
        out = op._apply(d, adjoint=True, gamma_inv=g)
    want = (g[:, None] if kind == "sensor" else g) * R.apply_adjoint(spec, d)
    assert R.rel_l2(out, want) <= 1e-12


@pytest.mark.parametrize("nrhs,nt", [(3, 16), (33, 16), (4, 15)])
def test_chunked_multi_rhs_host_path(btg, nrhs, nt):
    """Multi-RHS host calls (3M ZGEMM engine) stream column chunks as 2-D copies
    with the ZGEMM K-partials accumulated chunk by chunk: parity with the oracle
    and with the device-pointer path, epilogues included (ragged chunk, two RHS
    tiles at 33)."""
    import torch

    nd, nm = 20, 4500  # nt = 15: odd rows, the generic (unaligned) FFT path
    blocks, _, _ = R.random_problem(1600 + nrhs, nd, nm, nt)
    spec = R.setup_full(blocks)
    rng = np.random.default_rng(nrhs)
    M = rng.uniform(-1, 1, size=(nrhs, nm, nt))
    D = rng.uniform(-1, 1, size=(nrhs, nd, nt))
    gam = np.linspace(0.5, 2.0, nd)
    gm = rng.uniform(0.5, 2.0, size=(nm,))
    with btg.setup(blocks) as op:
        F = op.apply_forward(M)
        A = op.apply_adjoint(D)
        H = op.hessian_apply(M, alpha=0.2, reg="temporal-laplacian", gamma_inv=gam)
        Ag = op._apply(D, adjoint=True, gamma_inv=gm)
        F_dev = op.apply_forward(torch.from_numpy(M).cuda()).cpu().numpy()
        A_dev = op.apply_adjoint(torch.from_numpy(D).cuda()).cpu().numpy()
        assert np.array_equal(F, op.apply_forward(M))  # fixed chunk order: deterministic
    assert np.array_equal(A, A_dev)  # adjoint chunks partition the output columns
    assert R.rel_l2(F, F_dev) <= 1e-14
    for r in range(nrhs):
        assert R.rel_l2(F[r], R.apply_forward(spec, M[r])) <= 1e-12
        assert R.rel_l2(A[r], R.apply_adjoint(spec, D[r])) <= 1e-12
        assert R.rel_l2(H[r], R.gauss_newton_apply(spec, M[r], gam, 0.2, 1)) <= 1e-12
        assert R.rel_l2(Ag[r], gm[:, None] * R.apply_adjoint(spec, D[r])) <= 1e-12
