"""Parity of the CUDA path (through the C ABI) against the oracle — the
reference's own outputs (golden fixtures produced by oracle/_ref) and the numpy
restatement — plus the reference's known-answer / property tests replayed on
the GPU. Tolerance: relative L2 <= 1e-12 in FP64 (BASELINE.json north star),
<= 1e-5 for the FP32 F-hat mode; the reference's own per-test tolerances
(rel max-norm 1e-12 / 1e-11) where a test mirrors one of its cases."""

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


@pytest.fixture(scope="module")
def config_a(btg, golden_dir):
    g = np.load(golden_dir / "config_a_seed1.npz")
    nd, nm, nt = (int(x) for x in g["dims"])
    blocks, m, d = R.random_problem(int(g["seed"]), nd, nm, nt)
    op = btg.setup(blocks)
    yield g, blocks, m, d, op
    op.close()


def test_config_a_forward_adjoint_vs_reference(config_a):
    g, blocks, m, d, op = config_a
    assert R.rel_l2(op.apply_forward(m), g["fwd"]) <= TOL64
    assert R.rel_l2(op.apply_adjoint(d), g["adj"]) <= TOL64
    # and against the explicit dense block-Toeplitz matvec (configs[0] wording)
    D = R.dense_block_operator_soti(blocks)
    assert R.rel_l2(op.apply_forward(m).ravel(), D @ m.ravel()) <= TOL64
    assert R.rel_l2(op.apply_adjoint(d).ravel(), D.T @ d.ravel()) <= TOL64


def test_config_a_hessian_vs_reference(config_a):
    g, blocks, m, d, op = config_a
    assert R.rel_l2(op.hessian_apply(m), g["hess_a0"]) <= TOL64
    assert R.rel_l2(op.hessian_apply(m, alpha=0.1, reg="temporal-laplacian"), g["hess_lap"]) <= TOL64
    assert R.rel_l2(op.hessian_apply(m, alpha=0.25, reg="identity"), g["hess_id"]) <= TOL64
    # Gauss-Newton action with Gamma^-1 (pinned by composition of the reference's F and F*)
    assert R.rel_l2(op.hessian_apply(m, gamma_inv=g["gamma"]), g["gn_gamma"]) <= TOL64
    D = R.dense_block_operator_soti(blocks)
    w = np.repeat(g["gamma"], 64)
    assert R.rel_l2(op.hessian_apply(m, gamma_inv=g["gamma"]).ravel(), D.T @ (w * (D @ m.ravel()))) <= TOL64


def test_config_a_second_seed(btg, golden_dir):
    g = np.load(golden_dir / "config_a_seed20240901.npz")
    nd, nm, nt = (int(x) for x in g["dims"])
    blocks, m, d = R.random_problem(int(g["seed"]), nd, nm, nt)
    with btg.setup(blocks) as op:
        assert R.rel_l2(op.apply_forward(m), g["fwd"]) <= TOL64
        assert R.rel_l2(op.apply_adjoint(d), g["adj"]) <= TOL64


def test_gamma_per_sample(btg):
    blocks, m, d = R.random_problem(7, 6, 40, 24)
    gamma = R.ref_uniform(8, 6 * 24, 0.5, 2.0).reshape(6, 24)
    spec = R.setup_full(blocks)
    with btg.setup(blocks) as op:
        got = op.hessian_apply(m, alpha=0.3, reg="temporal-laplacian", gamma_inv=gamma)
        want = R.gauss_newton_apply(spec, m, gamma, 0.3, 1)
        assert R.rel_l2(got, want) <= TOL64


def test_spectrum_matches_reference_full_layout(btg, golden_dir):
    g = np.load(golden_dir / "small_case.npz")
    with btg.setup(g["blocks"]) as op:
        full = op.freq_blocks
        assert full.shape == g["spectrum"].shape
        scale = np.abs(g["spectrum"]).max()
        assert np.abs(full - g["spectrum"]).max() <= 1e-14 * scale
        assert R.rel_max_diff(op.apply_forward(g["m"]), g["fwd"]) < TOL64
        assert R.rel_max_diff(op.apply_adjoint(g["d"]), g["adj"]) < TOL64
        assert R.rel_max_diff(op.hessian_apply(g["m"], alpha=0.1), g["hess"]) < TOL64


def test_random_instances_vs_reference(btg, golden_dir):
    """test_block_operator.cpp:183-203 on the GPU: 40 ragged instances,
    N_t in 1..48 (odd, prime and composite FFT lengths), rel max-norm < 1e-11."""
    g = np.load(golden_dir / "random_instances.npz")
    rng = R.Mt19937_64(43)
    of = oa = 0
    for sensors, sources, steps in g["dims"]:
        rng.next_u64(3)
        blocks = rng.uniform(steps * sensors * sources, -1.0, 1.0).reshape(steps, sensors, sources)
        m = rng.uniform(sources * steps, -1.0, 1.0).reshape(sources, steps)
        d = rng.uniform(sensors * steps, -1.0, 1.0).reshape(sensors, steps)
        nfw, naj = sensors * steps, sources * steps
        with btg.setup(blocks) as op:
            got_f = op.apply_forward(m).ravel()
            got_a = op.apply_adjoint(d).ravel()
        assert R.rel_max_diff(got_f, g["fwd"][of : of + nfw]) < 1e-11, (sensors, sources, steps)
        assert R.rel_max_diff(got_a, g["adj"][oa : oa + naj]) < 1e-11, (sensors, sources, steps)
        of += nfw
        oa += naj


def test_identity_shift_zero_kats(btg):
    rng = R.Mt19937_64(31)
    eye = np.zeros((8, 3, 3))
    eye[0] = np.eye(3)
    m = rng.uniform(24, -1, 1).reshape(3, 8)
    with btg.setup(eye) as op:
        assert R.rel_max_diff(op.apply_forward(m), m) < TOL64
        assert R.rel_max_diff(op.apply_adjoint(m), m) < TOL64
    shift = np.zeros((6, 2, 2))
    shift[1] = np.eye(2)
    m = rng.uniform(12, -1, 1).reshape(2, 6)
    with btg.setup(shift) as op:
        dl = op.apply_forward(m)
        assert np.abs(dl[:, 0]).max() < 1e-12
        np.testing.assert_allclose(dl[:, 1:], m[:, :-1], rtol=1e-12, atol=1e-12)
        adv = op.apply_adjoint(m)
        assert np.abs(adv[:, -1]).max() < 1e-12
        np.testing.assert_allclose(adv[:, :-1], m[:, 1:], rtol=1e-12, atol=1e-12)
    with btg.setup(np.zeros((4, 2, 3))) as op:
        assert not op.spectrum().any()
        v = rng.uniform(12, -1, 1).reshape(3, 4)
        assert np.abs(op.hessian_apply(v)).max() < 1e-14
        np.testing.assert_allclose(op.hessian_apply(v, alpha=0.25), 0.25 * v, rtol=1e-14)


def test_causality_shift_equivariance_pairing(btg):
    """test_block_operator.cpp:205-264."""
    rng = R.Mt19937_64(47)
    blocks = rng.uniform(12 * 3 * 4, -1, 1).reshape(12, 3, 4)
    m = rng.uniform(4 * 12, -1, 1).reshape(4, 12)
    m[:, :5] = 0.0
    with btg.setup(blocks) as op:
        fast = op.apply_forward(m)
        assert np.abs(fast[:, :5]).max() <= 1e-12 * np.abs(m).max()
        m2 = rng.uniform(4 * 12, -1, 1).reshape(4, 12)
        dm = np.zeros_like(m2)
        dm[:, 1:] = m2[:, :-1]
        a, b = op.apply_forward(m2), op.apply_forward(dm)
        np.testing.assert_allclose(b[:, 1:], a[:, :-1], rtol=1e-11, atol=1e-12)
        d = rng.uniform(3 * 12, -1, 1).reshape(3, 12)
        lhs = np.vdot(op.apply_forward(m2), d)
        rhs = np.vdot(m2, op.apply_adjoint(d))
        assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), abs(rhs), 1.0)


def test_repeated_applies_are_bit_identical(btg):
    """test_block_operator.cpp:266-272 (fixed-order reductions, no atomics)."""
    blocks, m, d = R.random_problem(51, 40, 3000, 96)
    with btg.setup(blocks) as op:
        a = op.apply_forward(m)
        assert np.array_equal(a, op.apply_forward(m))
        b = op.apply_adjoint(d)
        assert np.array_equal(b, op.apply_adjoint(d))


def test_typed_errors(btg):
    """test_block_operator.cpp:274-282 / test_smoke.py:148-155."""
    eye = np.zeros((4, 2, 2))
    eye[0] = np.eye(2)
    with btg.setup(eye) as op:
        with pytest.raises(btg.DimensionError):
            op.apply_forward(np.zeros((3, 4)))
        with pytest.raises(ValueError):
            op.apply_adjoint(np.zeros((2, 5)))
        with pytest.raises(btg.Error):
            op.hessian_apply(np.zeros((2, 4)), reg="bogus")


def test_device_tensor_path_and_streams(btg):
    import torch

    blocks, m, d = R.random_problem(3, 5, 300, 50)
    spec = R.setup_full(blocks)
    bt = torch.from_numpy(blocks).cuda()
    with btg.setup(bt) as op:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            md = torch.from_numpy(m).cuda()
            out = op.apply_forward(md)
            back = op.apply_adjoint(out)
        s.synchronize()
        assert out.is_cuda and out.shape == (5, 50)
        assert R.rel_l2(out.cpu().numpy(), R.apply_forward(spec, m)) <= TOL64
        assert R.rel_l2(back.cpu().numpy(), R.hessian_apply(spec, m)) <= TOL64


def test_setup_rows_slabs_equal_full_setup_bitwise(btg):
    """Sharded setup reproduces the global F-hat bit-exactly
    (test_distributed.cpp:33-45): per-channel FFT arithmetic is independent of
    which slab / CTA batch a channel lands in."""
    blocks, m, _ = R.random_problem(9, 7, 33, 20)
    with btg.setup(blocks) as full:
        ref = full.spectrum()
    op = btg.create(7, 33, 20)
    for a, b in ((0, 3), (3, 4), (4, 7)):
        op.setup_rows(np.ascontiguousarray(blocks[:, a:b, :]), a, b)
    assert np.array_equal(op.spectrum(), ref)
    op.close()


def test_multiple_right_hand_sides(btg):
    blocks, m, d = R.random_problem(11, 6, 64, 32)
    spec = R.setup_full(blocks)
    rng = R.Mt19937_64(12)
    M = rng.uniform(4 * 64 * 32, -1, 1).reshape(4, 64, 32)
    Dv = rng.uniform(4 * 6 * 32, -1, 1).reshape(4, 6, 32)
    with btg.setup(blocks) as op:
        F = op.apply_forward(M)
        A = op.apply_adjoint(Dv)
        H = op.hessian_apply(M, alpha=0.2, reg="temporal-laplacian")
    for r in range(4):
        assert R.rel_l2(F[r], R.apply_forward(spec, M[r])) <= TOL64
        assert R.rel_l2(A[r], R.apply_adjoint(spec, Dv[r])) <= TOL64
        assert R.rel_l2(H[r], R.hessian_apply(spec, M[r], 0.2, 1)) <= TOL64


@pytest.mark.parametrize("dims", [(130, 300, 40, 33), (5, 77, 16, 2), (128, 256, 64, 32)])
def test_multi_rhs_dmma_zgemm(btg, dims, monkeypatch):
    """configs[3] shape class (ZGEMM on FP64 tensor cores): ragged N_d > 128
    (two row tiles), N_m not a multiple of the K chunk, nrhs > 32 (two RHS
    tiles); against the oracle and against the per-RHS GEMV path."""
    nd, nm, nt, nrhs = dims
    blocks, _, _ = R.random_problem(500 + nd, nd, nm, nt)
    spec = R.setup_full(blocks)
    rng = R.Mt19937_64(600 + nd)
    M = rng.uniform(nrhs * nm * nt, -1, 1).reshape(nrhs, nm, nt)
    Dv = rng.uniform(nrhs * nd * nt, -1, 1).reshape(nrhs, nd, nt)
    gam = np.linspace(0.5, 2.0, nd)
    with btg.setup(blocks) as op:
        F = op.apply_forward(M)
        A = op.apply_adjoint(Dv)
        H = op.hessian_apply(M, alpha=0.3, reg="temporal-laplacian", gamma_inv=gam)
    for r in range(nrhs):
        assert R.rel_l2(F[r], R.apply_forward(spec, M[r])) <= TOL64
        assert R.rel_l2(A[r], R.apply_adjoint(spec, Dv[r])) <= TOL64
        assert R.rel_l2(H[r], R.gauss_newton_apply(spec, M[r], gam, 0.3, 1)) <= TOL64
    monkeypatch.setenv("BTG_DISABLE_DMMA", "1")
    with btg.setup(blocks) as op:
        F2 = op.apply_forward(M)
    assert R.rel_l2(F, F2) <= 1e-14


@pytest.mark.parametrize("nt", [1, 2, 7, 64, 97, 125, 128, 256, 500, 512, 1000, 1001, 1024, 2000, 2048, 4096])
def test_fft_lengths(btg, nt):
    """Radix 2/4/8, 5 (N_t=1000 -> 2N_t=2000, configs[2]), 3, 7 and generic primes."""
    blocks, m, d = R.random_problem(100 + nt, 3, 9, nt)
    spec = R.setup_full(blocks)
    with btg.setup(blocks) as op:
        assert R.rel_l2(op.apply_forward(m), R.apply_forward(spec, m)) <= TOL64
        assert R.rel_l2(op.apply_adjoint(d), R.apply_adjoint(spec, d)) <= TOL64


def test_fp32_mode(btg):
    blocks, m, d = R.random_problem(13, 10, 500, 128)
    spec = R.setup_full(blocks)
    with btg.setup(blocks, precision=32) as op:
        assert R.rel_l2(op.apply_forward(m), R.apply_forward(spec, m)) <= TOL32
        assert R.rel_l2(op.apply_adjoint(d), R.apply_adjoint(spec, d)) <= TOL32
        assert R.rel_l2(op.hessian_apply(m, alpha=0.1), R.hessian_apply(spec, m, 0.1, 0)) <= TOL32
    # odd N_m exercises the 8-byte (unaligned row) load path
    blocks, m, d = R.random_problem(14, 5, 77, 30)
    spec = R.setup_full(blocks)
    with btg.setup(blocks, precision=32) as op:
        assert R.rel_l2(op.apply_forward(m), R.apply_forward(spec, m)) <= TOL32
        assert R.rel_l2(op.apply_adjoint(d), R.apply_adjoint(spec, d)) <= TOL32


@pytest.mark.slow
def test_baseline_shape_slice_vs_reference_build(btg):
    """configs[1] geometry (N_t=1024, N_d=100) on an N_m slice, against the
    reference build itself (oracle/_ref)."""
    from oracle import refcpu

    if not refcpu.available():
        pytest.skip("oracle/_ref not built")
    blocks, m, d = R.random_problem(2024, 100, 512, 1024)
    ref = refcpu.RefSpectralOperator(blocks)
    with btg.setup(blocks) as op:
        assert R.rel_l2(op.apply_forward(m), ref.apply_forward(m)) <= TOL64
        assert R.rel_l2(op.apply_adjoint(d), ref.apply_adjoint(d)) <= TOL64
        assert R.rel_l2(op.hessian_apply(m), ref.hessian_apply(m, 0.0, 0)) <= TOL64


def test_fast_and_generic_fft_paths_agree(btg, monkeypatch):
    """The compile-time-N register FFT (default for N_t in its plan table) and the
    generic shared-memory Stockham (BTG_DISABLE_FAST_FFT) give the same matvec."""
    blocks, m, d = R.random_problem(77, 5, 130, 1024)
    spec = R.setup_full(blocks)
    with btg.setup(blocks) as fast_op:
        f1, a1 = fast_op.apply_forward(m), fast_op.apply_adjoint(d)
        h1 = fast_op.hessian_apply(m, alpha=0.2, reg="temporal-laplacian", gamma_inv=np.linspace(0.5, 2, 5))
    monkeypatch.setenv("BTG_DISABLE_FAST_FFT", "1")
    with btg.setup(blocks) as gen_op:
        f2, a2 = gen_op.apply_forward(m), gen_op.apply_adjoint(d)
        h2 = gen_op.hessian_apply(m, alpha=0.2, reg="temporal-laplacian", gamma_inv=np.linspace(0.5, 2, 5))
    for got, other, want in ((f1, f2, R.apply_forward(spec, m)), (a1, a2, R.apply_adjoint(spec, d)),
                             (h1, h2, R.gauss_newton_apply(spec, m, np.linspace(0.5, 2, 5), 0.2, 1))):
        assert R.rel_l2(got, want) <= TOL64
        assert R.rel_l2(other, want) <= TOL64


def test_tma_gemv_path_matches(btg, monkeypatch):
    """The opt-in TMA-ring GEMV (BTG_GEMV_TMA=1) against the oracle, ragged shapes."""
    monkeypatch.setenv("BTG_GEMV_TMA", "1")
    for nd, nm, nt in ((13, 1500, 64), (100, 4096, 96), (3, 17, 20)):
        blocks, m, d = R.random_problem(900 + nm, nd, nm, nt)
        spec = R.setup_full(blocks)
        with btg.setup(blocks) as op:
            assert R.rel_l2(op.apply_forward(m), R.apply_forward(spec, m)) <= TOL64
            assert R.rel_l2(op.apply_adjoint(d), R.apply_adjoint(spec, d)) <= TOL64
            a = op.apply_forward(m)
            assert np.array_equal(a, op.apply_forward(m))


def test_misaligned_device_operands(btg):
    """Device operands that are 8- but not 16-byte aligned (a torch view at an
    odd storage offset) must take the generic C2R epilogue instead of faulting
    (the fast epilogue reads alpha R v and per-sample Gamma^-1 as 16-byte pairs)."""
    import torch

    blocks, m, d = R.random_problem(3, 6, 40, 64)
    spec = R.setup_full(blocks)
    op = btg.setup(blocks)
    try:
        nm, nt, nd = 40, 64, 6

        def odd_view(a):
            buf = torch.zeros(a.size + 1, dtype=torch.float64, device="cuda:0")
            v = buf[1:].view(a.shape)
            v.copy_(torch.from_numpy(a))
            assert v.data_ptr() % 16 == 8
            return v

        v = odd_view(m)
        got = op.hessian_apply(v, alpha=0.3, reg="temporal-laplacian").cpu().numpy()
        assert R.rel_l2(got, R.hessian_apply(spec, m, 0.3, 1)) <= TOL64
        g = np.random.default_rng(5).uniform(0.5, 2.0, size=(nd, nt))
        gv = odd_view(g)
        got = op.hessian_apply(torch.from_numpy(m).cuda(), gamma_inv=gv).cpu().numpy()
        assert R.rel_l2(got, R.gauss_newton_apply(spec, m, g, 0.0, 0)) <= TOL64
        got = op.apply_adjoint(torch.from_numpy(d).cuda(), reg_v=v, alpha=0.3, reg="identity").cpu().numpy()
        assert R.rel_l2(got, R.apply_adjoint(spec, d) + 0.3 * m) <= TOL64
        torch.cuda.synchronize()
    finally:
        op.close()
