"""More of the reference's own unit cases replayed on the GPU through the C ABI:
the pipeline counter model (proj/tests/test_block_operator.cpp:284-304), the
Hessian degenerate cases, dense normal matrix and SPD/symmetry checks
(proj/tests/test_inverse.cpp:81-132)."""

import math

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def btg():
    import paper_2407_13066_b200 as m

    return m


def test_pipeline_counters_follow_the_operation_model(btg):
    """test_block_operator.cpp:284-304 with the GPU's N_t+1 stored frequencies in
    the apply model: apply ops 8 N_d N_m NF, bytes 16 (N_d N_m + N_m
    + N_d) NF; pad / unpad / FFT op counts exactly the reference's."""
    sensors, sources, steps = 3, 5, 8
    nf, length = steps + 1, 2 * steps
    blocks, m, _ = R.random_problem(53, sensors, sources, steps)
    with btg.setup(blocks) as op:
        op.reset_counters()
        op.apply_forward(m)
        c = op.counters()
    assert c["apply"]["ops"] == 8.0 * sensors * sources * nf
    assert c["apply"]["bytes"] == 16.0 * (sensors * sources + sources + sensors) * nf
    assert c["pad"]["ops"] == 2.0 * sources * steps
    assert c["unpad"]["ops"] == 2.0 * sensors * steps
    assert c["forward_fft"]["ops"] == pytest.approx(sources * length * math.log2(length))
    assert c["inverse_fft"]["ops"] == pytest.approx(sensors * length * math.log2(length))
    assert c["launches"] >= 3


def test_hessian_degenerate_cases(btg):
    zeros = np.zeros((4, 2, 3))
    v = R.ref_uniform(205, 3 * 4).reshape(3, 4)
    with btg.setup(zeros) as op:
        assert np.abs(op.hessian_apply(v)).max() < 1e-14
        hv = op.hessian_apply(v, alpha=0.25, reg="identity")
    assert np.allclose(hv, 0.25 * v, rtol=1e-14, atol=0)


def test_hessian_matches_dense_normal_matrix(btg):
    blocks, _, _ = R.random_problem(209, 3, 4, 8)
    v = R.ref_uniform(210, 4 * 8).reshape(4, 8)
    D = R.dense_block_operator_soti(blocks)
    H = D.T @ D + 0.1 * np.eye(32)
    with btg.setup(blocks) as op:
        hv = op.hessian_apply(v, alpha=0.1, reg="identity")
    assert R.rel_max_diff(hv.ravel(), H @ v.ravel()) < 1e-11


def test_hessian_symmetric_positive_definite(btg):
    blocks, _, _ = R.random_problem(211, 2, 3, 6)
    rng = R.Mt19937_64(212)
    with btg.setup(blocks) as op:
        for _ in range(100):
            v = rng.uniform(18, -1, 1).reshape(3, 6)
            w = rng.uniform(18, -1, 1).reshape(3, 6)
            hv = op.hessian_apply(v, alpha=0.2, reg="temporal-laplacian")
            hw = op.hessian_apply(w, alpha=0.2, reg="temporal-laplacian")
            vw, wv = float(hv.ravel() @ w.ravel()), float(v.ravel() @ hw.ravel())
            assert abs(vw - wv) <= 1e-10 * max(abs(vw), abs(wv), 1.0)
            assert float(hv.ravel() @ v.ravel()) > 0.0
