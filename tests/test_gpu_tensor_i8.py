"""Parity of the opt-in multi-RHS Fourier step on tcgen05 int8 tensor cores
(Ozaki splitting, BTG_TENSOR_I8=1, csrc/btg_ozaki.cu) against the oracle and
against the DMMA ZGEMM path. FP64 tolerance: relative L2 <= 1e-12 (north star)."""

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu

TOL64 = 1e-12


@pytest.fixture(scope="module")
def btg():
    import paper_2407_13066_b200 as m

    return m


@pytest.mark.parametrize("dims", [(8, 64, 16, 2), (130, 300, 40, 33), (5, 77, 16, 9), (128, 2100, 32, 32),
                                  (300, 1100, 8, 17)])
def test_tensor_i8_multi_rhs(btg, dims, monkeypatch):
    """Ragged N_d (several 128-row tiles in the adjoint), N_m across 1024-wide
    scale blocks, nrhs not a multiple of 8 and > 32 (two RHS passes)."""
    nd, nm, nt, nrhs = dims
    blocks, _, _ = R.random_problem(700 + nd, nd, nm, nt)
    spec = R.setup_full(blocks)
    rng = R.Mt19937_64(800 + nd)
    M = rng.uniform(nrhs * nm * nt, -1, 1).reshape(nrhs, nm, nt)
    Dv = rng.uniform(nrhs * nd * nt, -1, 1).reshape(nrhs, nd, nt)
    gam = np.linspace(0.5, 2.0, nd)
    monkeypatch.setenv("BTG_TENSOR_I8", "1")
    with btg.setup(blocks) as op:
        F = op.apply_forward(M)
        A = op.apply_adjoint(Dv)
        H = op.hessian_apply(M, alpha=0.3, reg="temporal-laplacian", gamma_inv=gam)
        assert np.array_equal(F, op.apply_forward(M))  # deterministic repeats
    for r in range(nrhs):
        assert R.rel_l2(F[r], R.apply_forward(spec, M[r])) <= TOL64
        assert R.rel_l2(A[r], R.apply_adjoint(spec, Dv[r])) <= TOL64
        assert R.rel_l2(H[r], R.gauss_newton_apply(spec, M[r], gam, 0.3, 1)) <= TOL64


def test_tensor_i8_wide_dynamic_range(btg, monkeypatch):
    """Entries spanning many binades inside one scale block: the block-max
    splitting must still meet 1e-12 in relative L2 of the output."""
    nd, nm, nt, nrhs = 16, 512, 16, 4
    blocks, _, _ = R.random_problem(901, nd, nm, nt)
    rng = np.random.default_rng(5)
    blocks = blocks * np.exp2(rng.integers(-20, 4, size=blocks.shape))
    spec = R.setup_full(blocks)
    M = rng.uniform(-1, 1, size=(nrhs, nm, nt)) * np.exp2(rng.integers(-10, 10, size=(nrhs, nm, 1)))
    monkeypatch.setenv("BTG_TENSOR_I8", "1")
    with btg.setup(blocks) as op:
        F = op.apply_forward(M)
    for r in range(nrhs):
        assert R.rel_l2(F[r], R.apply_forward(spec, M[r])) <= TOL64


def test_engine_switch_on_one_handle(btg):
    """btg_set_multi_rhs_engine: the same handle alternates DMMA and tcgen05
    int8 engines; both meet the FP64 bar against the oracle."""
    nd, nm, nt, nrhs = 40, 1500, 24, 5
    blocks, _, _ = R.random_problem(950, nd, nm, nt)
    spec = R.setup_full(blocks)
    M = R.Mt19937_64(951).uniform(nrhs * nm * nt, -1, 1).reshape(nrhs, nm, nt)
    with btg.setup(blocks) as op:
        F_dmma = op.apply_forward(M)
        op.set_multi_rhs_engine("tensor_i8")
        F_i8 = op.apply_forward(M)
        A_i8 = op.apply_adjoint(F_i8)
        op.set_multi_rhs_engine("dmma")
        A_dmma = op.apply_adjoint(F_dmma)
        with pytest.raises(ValueError):
            op.set_multi_rhs_engine("tf32")
    for r in range(nrhs):
        want = R.apply_forward(spec, M[r])
        assert R.rel_l2(F_dmma[r], want) <= TOL64
        assert R.rel_l2(F_i8[r], want) <= TOL64
        assert R.rel_l2(A_i8[r], A_dmma[r]) <= TOL64


@pytest.mark.parametrize("dims", [(130, 2048, 64, 9), (40, 1104, 256, 32), (12, 3076, 1024, 5)])
def test_fused_block_max_matches_scale_pass(btg, dims, monkeypatch):
    """Lengths with a fast R2C plan: the x-hat block maxima come out of the R2C
    epilogue (R2CBlockMax) instead of a separate pass; the exponents are the same
    exact maxima, so the results are bit-identical to the scale pass and meet the
    FP64 bar against the oracle."""
    nd, nm, nt, nrhs = dims
    blocks, _, _ = R.random_problem(1200 + nt, nd, nm, nt)
    spec = R.setup_full(blocks)
    M = R.Mt19937_64(1300 + nt).uniform(nrhs * nm * nt, -1, 1).reshape(nrhs, nm, nt)
    with btg.setup(blocks) as op:
        op.set_multi_rhs_engine("tensor_i8")
        fused = op.apply_forward(M)
        monkeypatch.setenv("BTG_OZ_SCALE_PASS", "1")
        separate = op.apply_forward(M)
    assert np.array_equal(fused, separate)
    for r in range(nrhs):
        assert R.rel_l2(fused[r], R.apply_forward(spec, M[r])) <= TOL64
