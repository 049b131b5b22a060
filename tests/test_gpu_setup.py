"""Setup (Alg. 1, block_operator.cpp:178-205) on the transposed path: for FP64
and an N_t with a compile-time FFT plan, each TOSI slab is transposed to SOTI
rows in a bounded device buffer and run through the vector R2C
(btg_setup_rows). The spectrum matches the oracle and the generic strided path
(BTG_SETUP_GENERIC=1), and each channel's transform is placement-independent
(test_distributed.cpp:33-45's serial == sharded property at a fast-plan size)."""

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def btg():
    import paper_2407_13066_b200 as m

    return m


@pytest.mark.parametrize("nt,nd,nm", [(1024, 3, 301), (64, 5, 77), (1000, 2, 45)])
def test_transposed_setup_matches_oracle_and_generic(btg, monkeypatch, nt, nd, nm):
    import torch

    blocks, _, _ = R.random_problem(nt + nd, nd, nm, nt)
    want = R.setup_full(blocks)[: nt + 1]
    got = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("BTG_SETUP_GENERIC", mode)
        with btg.setup(blocks) as op:  # host slabs
            got[mode] = op.spectrum()
        with btg.setup(torch.from_numpy(blocks).cuda()) as op:  # device slab
            assert np.array_equal(op.spectrum(), got[mode])
    monkeypatch.delenv("BTG_SETUP_GENERIC", raising=False)
    for mode in ("0", "1"):
        assert R.rel_l2(got[mode], want) <= 1e-14
    assert R.rel_l2(got["0"], got["1"]) <= 1e-14


def test_transposed_setup_placement_independent_at_scale(btg):
    """262144 channels in one slab (the non-TMA vector R2C) against four 65536-
    channel row slabs (the TMA R2C): the same F-hat bits, seen through F m."""
    import torch

    nt, nd, nm = 1024, 4, 65536
    g = torch.Generator(device="cuda").manual_seed(5)
    blocks = torch.rand((nt, nd, nm), dtype=torch.float64, device="cuda", generator=g) - 0.5
    m = torch.rand((nm, nt), dtype=torch.float64, device="cuda", generator=g) - 0.5
    with btg.setup(blocks) as full:
        d_full = full.apply_forward(m)
        op = btg.create(nd, nm, nt)
        try:
            for i in range(nd):
                op.setup_rows(blocks[:, i : i + 1, :].contiguous(), i, i + 1)
            d_rows = op.apply_forward(m)
        finally:
            op.close()
    assert torch.equal(d_full, d_rows)
    # and one sensor row against the oracle (numpy FFT of the host copy)
    b0 = blocks[:, :1, :4096].cpu().numpy()
    spec = R.setup_full(b0)
    with btg.setup(np.ascontiguousarray(b0)) as small:
        assert R.rel_l2(small.spectrum(), spec[: nt + 1]) <= 1e-14


@pytest.mark.parametrize("nt,nd,nm", [(1024, 3, 301), (4096, 2, 33)])
def test_transposed_setup_fp32_fhat(btg, monkeypatch, nt, nd, nm):
    """FP32 F-hat: the complex128 vector-R2C block rounded to complex64
    (k_spec_to_f32) — within FP32 rounding of the oracle and of the generic
    strided path (whose FP64 sums differ from the vector R2C's in the last bits,
    so an element may round to the neighbouring float)."""
    blocks, _, _ = R.random_problem(nt + 3 * nd, nd, nm, nt)
    want = R.setup_full(blocks)[: nt + 1]
    got = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("BTG_SETUP_GENERIC", mode)
        with btg.setup(blocks, precision=32) as op:
            got[mode] = op.spectrum()
    monkeypatch.delenv("BTG_SETUP_GENERIC", raising=False)
    for mode in ("0", "1"):
        assert R.rel_l2(got[mode], want) <= 1e-7
    assert R.rel_l2(got["0"], got["1"]) <= 1e-7
