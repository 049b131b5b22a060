"""Pin the oracle before trusting it (CPU only).

* the numpy restatement (oracle/restate.py) against the golden vectors the
  reference itself produced (tests/golden/make_golden.py via oracle/_ref);
* the restatement against the reference's own known-answer and property tests
  (test_block_operator.cpp, test_inverse.cpp, test_distributed.cpp);
* the RNG port against std::mt19937_64 inside the reference build.
"""

import numpy as np
import pytest

from oracle import restate as R

TOL = 1e-12


def test_rng_port_matches_reference_stream_fingerprint(golden_dir):
    g = np.load(golden_dir / "config_a_seed1.npz")
    nd, nm, nt = g["dims"]
    blocks, m, d = R.random_problem(int(g["seed"]), nd, nm, nt)
    fp = np.array([blocks.sum(), m.sum(), d.sum(), blocks.ravel()[-1], m.ravel()[-1], d.ravel()[-1]])
    np.testing.assert_array_equal(fp, g["fingerprint"])


def test_rng_known_values():
    # std::mt19937_64 default-seed 10000th output is 9981545732273789042 (C++ standard 26.5.5)
    rng = R.Mt19937_64(5489)
    assert int(rng.next_u64(10000)[-1]) == 9981545732273789042


@pytest.mark.parametrize("name", ["config_a_seed1.npz", "config_a_seed20240901.npz"])
def test_restatement_matches_reference_config_a(golden_dir, name):
    g = np.load(golden_dir / name)
    nd, nm, nt = (int(x) for x in g["dims"])
    blocks, m, d = R.random_problem(int(g["seed"]), nd, nm, nt)
    spec = R.setup_full(blocks)
    assert R.rel_l2(R.apply_forward(spec, m), g["fwd"]) < TOL
    assert R.rel_l2(R.apply_adjoint(spec, d), g["adj"]) < TOL
    if "hess_lap" in g:
        assert R.rel_l2(R.hessian_apply(spec, m, 0.0, 0), g["hess_a0"]) < TOL
        assert R.rel_l2(R.hessian_apply(spec, m, 0.1, 1), g["hess_lap"]) < TOL
        assert R.rel_l2(R.hessian_apply(spec, m, 0.25, 0), g["hess_id"]) < TOL
        assert R.rel_l2(R.gauss_newton_apply(spec, m, g["gamma"]), g["gn_gamma"]) < TOL
        assert R.rel_l2(R.naive_apply_forward(blocks, m), g["naive_fwd"]) < TOL


def test_restatement_matches_reference_small_case_and_spectrum(golden_dir):
    g = np.load(golden_dir / "small_case.npz")
    spec = R.setup_full(g["blocks"])
    scale = np.abs(g["spectrum"]).max()
    assert np.abs(spec - g["spectrum"]).max() <= 1e-14 * scale
    assert R.rel_max_diff(R.apply_forward(spec, g["m"]), g["fwd"]) < TOL
    assert R.rel_max_diff(R.apply_adjoint(spec, g["d"]), g["adj"]) < TOL
    assert R.rel_max_diff(R.hessian_apply(spec, g["m"], 0.1, 0), g["hess"]) < TOL


def test_restatement_random_instances(golden_dir):
    """test_block_operator.cpp:183-203 (40 trials, rel max-norm < 1e-11)."""
    g = np.load(golden_dir / "random_instances.npz")
    rng = R.Mt19937_64(43)
    of = oa = 0
    for sensors, sources, steps in g["dims"]:
        # consume the same three integer draws the reference made
        rng.next_u64(3)
        blocks = rng.uniform(steps * sensors * sources, -1.0, 1.0).reshape(steps, sensors, sources)
        m = rng.uniform(sources * steps, -1.0, 1.0).reshape(sources, steps)
        d = rng.uniform(sensors * steps, -1.0, 1.0).reshape(sensors, steps)
        spec = R.setup_full(blocks)
        nfw, naj = sensors * steps, sources * steps
        assert R.rel_max_diff(R.apply_forward(spec, m).ravel(), g["fwd"][of : of + nfw]) < 1e-11
        assert R.rel_max_diff(R.apply_adjoint(spec, d).ravel(), g["adj"][oa : oa + naj]) < 1e-11
        assert R.rel_max_diff(g["naive_fwd"][of : of + nfw], g["fwd"][of : of + nfw]) < 1e-11
        of += nfw
        oa += naj
    assert of == g["fwd"].size and oa == g["adj"].size


def test_kat_identity_and_shift():
    """test_block_operator.cpp:88-115."""
    rng = R.Mt19937_64(31)
    eye = np.zeros((8, 3, 3))
    eye[0] = np.eye(3)
    spec = R.setup_full(eye)
    m = rng.uniform(3 * 8, -1, 1).reshape(3, 8)
    assert R.rel_max_diff(R.apply_forward(spec, m), m) < TOL
    assert R.rel_max_diff(R.apply_adjoint(spec, m), m) < TOL
    shift = np.zeros((6, 2, 2))
    shift[1] = np.eye(2)
    spec = R.setup_full(shift)
    m = rng.uniform(2 * 6, -1, 1).reshape(2, 6)
    delayed = R.apply_forward(spec, m)
    np.testing.assert_allclose(delayed[:, 1:], m[:, :-1], rtol=1e-12, atol=1e-12)
    assert np.abs(delayed[:, 0]).max() < 1e-12
    adv = R.apply_adjoint(spec, m)
    np.testing.assert_allclose(adv[:, :-1], m[:, 1:], rtol=1e-12, atol=1e-12)


def test_conjugate_symmetry_and_dense():
    """test_block_operator.cpp:73-86, 126-140 and tests/oracles.cpp dense oracle."""
    rng = R.Mt19937_64(23)
    blocks = rng.uniform(5 * 3 * 2, -1, 1).reshape(5, 3, 2)
    spec = R.setup_full(blocks)
    L = spec.shape[0]
    sym = np.conj(spec[(L - np.arange(L)) % L])
    assert np.abs(spec - sym).max() <= 1e-13 * np.abs(spec).max()
    D = R.dense_block_operator_soti(blocks)
    m = rng.uniform(2 * 5, -1, 1).reshape(2, 5)
    d = rng.uniform(3 * 5, -1, 1).reshape(3, 5)
    assert R.rel_max_diff(R.apply_forward(spec, m).ravel(), D @ m.ravel()) < TOL
    assert R.rel_max_diff(R.apply_adjoint(spec, d).ravel(), D.T @ d.ravel()) < TOL


def test_hessian_dense_normal_matrix():
    """test_inverse.cpp:100-117: H = F^T F + alpha I vs dense."""
    rng = R.Mt19937_64(209)
    blocks = rng.uniform(8 * 3 * 4, -1, 1).reshape(8, 3, 4)
    spec = R.setup_full(blocks)
    F = R.dense_block_operator_soti(blocks)
    H = F.T @ F + 0.1 * np.eye(32)
    v = rng.uniform(4 * 8, -1, 1).reshape(4, 8)
    assert R.rel_max_diff(R.hessian_apply(spec, v, 0.1, 0).ravel(), H @ v.ravel()) < 1e-11


def test_distributed_restatement_matches_reference(golden_dir):
    """test_smoke.py:68-78 grids and the ceiling partition (distributed.cpp:145-175)."""
    g = np.load(golden_dir / "distributed_case.npz")
    blocks, m, d = R.random_problem(5, 5, 7, 12)
    spec = R.setup_full(blocks)
    for grid in ("1x4", "2x2", "4x1", "2x3"):
        r, c = map(int, grid.split("x"))
        assert [tuple(b) for b in g[f"bounds_{grid}"]] == R.partition_bounds(5, 7, r, c)
        assert R.rel_max_diff(R.apply_forward(spec, m), g[f"fwd_{grid}"]) < TOL
        assert R.rel_max_diff(R.apply_adjoint(spec, d), g[f"adj_{grid}"]) < TOL
    with pytest.raises(ValueError):
        R.partition_bounds(2, 3, 3, 1)
    with pytest.raises(ValueError):
        R.partition_bounds(2, 3, 1, 4)


def test_tree_reduce_order():
    """distributed.cpp:38-47: ((v0+v1)+(v2+v3))+v4."""
    vals = [np.array([1e16]), np.array([1.0]), np.array([-1e16]), np.array([1.0]), np.array([3.0])]
    expected = ((vals[0] + vals[1]) + (vals[2] + vals[3])) + vals[4]
    np.testing.assert_array_equal(R.tree_reduce(vals), expected)


def test_reference_build_self_verification():
    from oracle import refcpu

    if not refcpu.available():
        pytest.skip("oracle/_ref not built")
    ok, report = refcpu.verify(20240901)
    assert ok, report
    assert report.count("[PASS]") == 12


def test_reference_ewp_fixture_matches_restatement(golden_dir):
    """The reference's EWP backend (block_operator.cpp:345-421, tests/golden/ewp_case.npz)
    computes the same map as the FFT pipeline restated here."""
    g = np.load(golden_dir / "ewp_case.npz")
    for tag in ("a", "r"):
        nd, nm, nt = (int(x) for x in g[f"{tag}_dims"])
        blocks, m, d = R.random_problem(int(g[f"{tag}_seed"]), nd, nm, nt)
        fp = [float(np.sum(a)) for a in (blocks, m, d)] + [float(a.ravel()[-1]) for a in (blocks, m, d)]
        assert np.array_equal(np.array(fp), g[f"{tag}_fingerprint"])  # the RNG port drew the same inputs
        spec = R.setup_full(blocks)
        assert R.rel_l2(g[f"{tag}_fwd"], R.apply_forward(spec, m)) <= 1e-13
        assert R.rel_l2(g[f"{tag}_adj"], R.apply_adjoint(spec, d)) <= 1e-13
