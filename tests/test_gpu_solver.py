"""Device-resident CG (btg_cg_solve) and objective (btg_objective) against the
reference's own cg_solve / objective_eval (oracle/_ref, inverse.cpp:93-156)
and the reference's solver tests (test_smoke.py:102-114, test_inverse.cpp)."""

import numpy as np
import pytest

from oracle import refcpu
from oracle import restate as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def btg():
    import paper_2407_13066_b200 as m

    return m


needs_ref = pytest.mark.skipif(not refcpu.available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("reg,precond,alpha", [("identity", False, 0.05), ("temporal-laplacian", False, 0.5),
                                               ("temporal-laplacian", True, 0.05)])
def test_cg_matches_reference_cg(btg, reg, precond, alpha):
    blocks, m_true, _ = R.random_problem(71, 6, 20, 32)
    kind = 0 if reg == "identity" else 1
    ref = refcpu.RefSpectralOperator(blocks)
    d_obs = ref.apply_forward(m_true)
    rhs = ref.apply_adjoint(d_obs)
    x_ref, it_ref, res_ref, conv_ref = ref.cg_solve(rhs, alpha, kind, tol=1e-10, maxiter=2000,
                                                    precondition=precond)
    assert conv_ref
    with btg.setup(blocks) as op:
        x, it, res, conv = btg.cg_solve_op(op, rhs, alpha=alpha, reg=reg, tol=1e-10, maxiter=2000,
                                           precondition=precond)
        assert conv
        # long CG runs drift from exact arithmetic differently under different
        # (both deterministic) summation orders: counts agree to within 10 %
        assert abs(it - it_ref) <= max(2, it_ref // 10)
        assert res <= 1e-10
        # both iterates solve H x = rhs to 1e-10 relative residual; their gap is
        # bounded by cond(H) * tol (the Laplacian case without R^-1 is the worst)
        assert R.rel_l2(x, x_ref) <= 1e-6
        # the solution satisfies the normal equations
        hx = op.hessian_apply(x, alpha=alpha, reg=reg)
        assert R.rel_l2(hx, rhs) <= 1e-9
        # objective matches the reference's objective_eval
        want = ref.objective(x, d_obs, alpha, kind)
        assert abs(btg.objective_eval(op, x, d_obs, alpha=alpha, reg=reg) - want) <= 1e-12 * max(1.0, abs(want))


def test_cg_recovers_noiseless_data_like_reference_smoke(btg):
    """test_smoke.py:102-114 replayed through the reference binding's signature."""
    rng = np.random.default_rng(7)
    blocks = rng.uniform(-1.0, 1.0, size=(8, 3, 3))
    m_true = rng.uniform(-1.0, 1.0, size=(3, 8))
    with btg.setup(blocks) as op:
        d_obs = op.apply_forward(m_true)
    m, iterations, residual, converged = btg.cg_solve(blocks, d_obs, alpha=1e-8, tol=1e-12, maxiter=2000)
    assert converged
    assert iterations >= 1
    with btg.setup(blocks) as op:
        misfit = np.linalg.norm(op.apply_forward(m) - d_obs) / np.linalg.norm(d_obs)
    assert misfit <= 1e-6
    assert residual <= 1e-12


def test_cg_zero_rhs_and_solver_error(btg):
    blocks, _, _ = R.random_problem(3, 2, 4, 8)
    with btg.setup(blocks) as op:
        x, it, res, conv = btg.cg_solve_op(op, np.zeros((4, 8)), alpha=0.1)
        assert conv and it == 0 and not x.any()
        # alpha < 0 on the zero operator: H = alpha I is negative definite -> SolverError
    with btg.setup(np.zeros((8, 2, 4))) as op:
        with pytest.raises(btg.SolverError):
            btg.cg_solve_op(op, np.ones((4, 8)), alpha=-1.0)


def test_cg_device_tensors_and_gamma(btg):
    import torch

    blocks, m_true, _ = R.random_problem(72, 5, 30, 40)
    gam = np.linspace(0.5, 2.0, 5)
    spec = R.setup_full(blocks)
    d_obs = R.apply_forward(spec, m_true)
    rhs = R.apply_adjoint(spec, gam[:, None] * d_obs)
    with btg.setup(blocks) as op:
        x, it, res, conv = btg.cg_solve_op(op, torch.from_numpy(rhs).cuda(), alpha=0.02, tol=1e-11,
                                           maxiter=800, gamma_inv=torch.from_numpy(gam).cuda())
        assert conv
        x = x.cpu().numpy()
    want = R.gauss_newton_apply(spec, x, gam, 0.02, 0)
    assert R.rel_l2(want, rhs) <= 1e-9


def test_cg_solve_with_grid_matches_single_worker(btg):
    """The reference binding accepts any RxC grid (bindings.cpp:229-249): rhs from
    distributed_adjoint over a Partition, same Hessian."""
    rng = np.random.default_rng(11)
    blocks = rng.uniform(-1.0, 1.0, size=(16, 4, 6))
    d_obs = rng.uniform(-1.0, 1.0, size=(4, 16))
    m1, it1, res1, c1 = btg.cg_solve(blocks, d_obs, alpha=0.05, tol=1e-12, maxiter=500)
    m2, it2, res2, c2 = btg.cg_solve(blocks, d_obs, alpha=0.05, tol=1e-12, maxiter=500, grid="2x3")
    assert c1 and c2
    assert np.linalg.norm(m1 - m2) <= 1e-10 * np.linalg.norm(m1)


@pytest.mark.parametrize("reg,precond,gamma", [("identity", False, False), ("temporal-laplacian", True, True),
                                               ("temporal-laplacian", False, True)])
def test_cg_graph_loop_matches_host_loop_bitwise(btg, monkeypatch, reg, precond, gamma):
    """The default solver runs the whole iteration loop as one CUDA graph WHILE
    node with the scalars on the device; BTG_CG_HOST_LOOP=1 selects the loop
    that reads pHp and ||r||^2 back every iteration. Same operations, same
    fixed-grid reductions: identical iterates, residuals and counts."""
    blocks, m_true, _ = R.random_problem(73, 6, 24, 48)
    spec = R.setup_full(blocks)
    rhs = R.apply_adjoint(spec, R.apply_forward(spec, m_true))
    gam = np.linspace(0.5, 2.0, 6) if gamma else None
    with btg.setup(blocks) as op:
        outs = []
        for host in (False, True):
            if host:
                monkeypatch.setenv("BTG_CG_HOST_LOOP", "1")
            else:
                monkeypatch.delenv("BTG_CG_HOST_LOOP", raising=False)
            outs.append(btg.cg_solve_op(op, rhs, alpha=0.03, reg=reg, tol=1e-10, maxiter=3000,
                                        precondition=precond, gamma_inv=gam))
        monkeypatch.delenv("BTG_CG_HOST_LOOP", raising=False)
        (xg, itg, resg, cg), (xh, ith, resh, ch) = outs
        assert cg == ch
        assert itg == ith
        assert resg == resh
        assert np.array_equal(xg, xh)
        # an iteration cap stops both loops at the same iterate
        x5g, it5g, res5g, c5g = btg.cg_solve_op(op, rhs, alpha=0.03, reg=reg, tol=1e-30, maxiter=5,
                                                precondition=precond, gamma_inv=gam)
        monkeypatch.setenv("BTG_CG_HOST_LOOP", "1")
        x5h, it5h, res5h, c5h = btg.cg_solve_op(op, rhs, alpha=0.03, reg=reg, tol=1e-30, maxiter=5,
                                                precondition=precond, gamma_inv=gam)
        monkeypatch.delenv("BTG_CG_HOST_LOOP", raising=False)
        assert it5g == it5h == 5 and not c5g and not c5h
        assert res5g == res5h and np.array_equal(x5g, x5h)
