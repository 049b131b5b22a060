"""Long horizons: N_t beyond the shared-memory two-buffer transform.

The paper's largest runs use N_t = 10000 time steps; the reference's FFT
handles any length (its Bluestein path, fft.cpp). Here N_t = 8192 and 10000
take the register-resident compile-time plans for vector transforms, and every
length whose generic transform does not fit shared memory (setup, FP32 setup,
lengths without a plan such as 7000 or 6561 = 3^8) runs the generic kernels on
a global scratch. Same FP64 tolerance as everywhere: rel L2 <= 1e-12.
"""

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-5


@pytest.fixture(scope="module")
def btg():
    import paper_2407_13066_b200 as m

    return m


@pytest.mark.parametrize("nt", [6561, 7000, 8192, 10000])
def test_long_horizon_forward_adjoint_hessian(btg, nt):
    blocks, m, d = R.random_problem(7 + nt, 3, 5, nt)
    spec = R.setup_full(blocks)
    with btg.setup(blocks) as op:
        assert R.rel_l2(op.apply_forward(m), R.apply_forward(spec, m)) <= TOL64
        assert R.rel_l2(op.apply_adjoint(d), R.apply_adjoint(spec, d)) <= TOL64
        assert R.rel_l2(op.hessian_apply(m, alpha=0.1, reg=1),
                        R.hessian_apply(spec, m, 0.1, 1)) <= TOL64
        # the stored half spectrum itself (setup ran on the global scratch)
        half = op.spectrum()
        assert R.rel_l2(half, spec[: nt + 1]) <= TOL64


@pytest.mark.parametrize("nt", [8192, 10000])
def test_long_horizon_fast_matches_generic(btg, nt, monkeypatch):
    blocks, m, d = R.random_problem(11 + nt, 2, 4, nt)
    with btg.setup(blocks) as op:
        fast_f, fast_a = op.apply_forward(m), op.apply_adjoint(d)
    monkeypatch.setenv("BTG_DISABLE_FAST_FFT", "1")
    with btg.setup(blocks) as op:
        gen_f, gen_a = op.apply_forward(m), op.apply_adjoint(d)
    assert R.rel_l2(fast_f, gen_f) <= TOL64
    assert R.rel_l2(fast_a, gen_a) <= TOL64


def test_long_horizon_fp32(btg):
    nt = 10000
    blocks, m, d = R.random_problem(5, 3, 6, nt)
    spec = R.setup_full(blocks)
    with btg.setup(blocks, precision=32) as op:
        assert R.rel_l2(op.apply_forward(m), R.apply_forward(spec, m)) <= TOL32
        assert R.rel_l2(op.apply_adjoint(d), R.apply_adjoint(spec, d)) <= TOL32


def test_long_horizon_multi_rhs(btg):
    """Several right-hand sides (the DMMA ZGEMM path) at N_t = 8192."""
    nt, k = 8192, 3
    blocks, _, _ = R.random_problem(3, 4, 6, nt)
    spec = R.setup_full(blocks)
    rng = np.random.default_rng(0)
    ms = rng.standard_normal((k, 6, nt))
    with btg.setup(blocks) as op:
        out = op.apply_forward(ms)
        for r in range(k):
            assert R.rel_l2(out[r], R.apply_forward(spec, ms[r])) <= TOL64


def test_horizon_beyond_grid_y_limit(btg):
    """N_t + 1 > 65535 frequencies: the Fourier-space kernels run in frequency
    batches (grid.y limit), single- and multi-RHS."""
    nt = 70000
    blocks, m, d = R.random_problem(9, 2, 3, nt)
    spec = R.setup_full(blocks)
    with btg.setup(blocks) as op:
        assert R.rel_l2(op.apply_forward(m), R.apply_forward(spec, m)) <= TOL64
        assert R.rel_l2(op.apply_adjoint(d), R.apply_adjoint(spec, d)) <= TOL64
        ms = np.stack([m, 2.0 * m[::-1]])
        out = op.apply_forward(ms)
        for r in range(2):
            assert R.rel_l2(out[r], R.apply_forward(spec, ms[r])) <= TOL64
        ds = np.stack([d, -d])
        outa = op.apply_adjoint(ds)
        for r in range(2):
            assert R.rel_l2(outa[r], R.apply_adjoint(spec, ds[r])) <= TOL64
