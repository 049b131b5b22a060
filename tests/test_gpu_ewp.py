"""EWP backend (the reference's Appendix A formulation, block_operator.cpp:345-421)
on the GPU: channel-major spectrum + element-wise products, against the
reference's own EWP outputs (tests/golden/ewp_case.npz, produced by oracle/_ref)
and the FFT backend. FP64 tolerance: relative L2 <= 1e-12."""

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu

TOL64 = 1e-12


@pytest.fixture(scope="module")
def btg():
    import paper_2407_13066_b200 as m

    return m


@pytest.mark.parametrize("tag", ["a", "r"])
def test_ewp_matches_reference_ewp(btg, golden_dir, tag):
    g = np.load(golden_dir / "ewp_case.npz")
    nd, nm, nt = (int(x) for x in g[f"{tag}_dims"])
    blocks, m, d = R.random_problem(int(g[f"{tag}_seed"]), nd, nm, nt)
    with btg.setup(blocks, keep_channel_layout=True) as op:
        assert op.has_channel_layout
        assert R.rel_l2(op.apply_forward_ewp(m), g[f"{tag}_fwd"]) <= TOL64
        assert R.rel_l2(op.apply_adjoint_ewp(d), g[f"{tag}_adj"]) <= TOL64
        # same spectrum, other loop order: the FFT backend agrees
        assert R.rel_l2(op.apply_forward_ewp(m), op.apply_forward(m)) <= 1e-14


def test_ewp_requires_channel_layout(btg):
    blocks, m, _ = R.random_problem(3, 2, 5, 8)
    with btg.setup(blocks) as op:
        assert not op.has_channel_layout
        with pytest.raises(RuntimeError, match="channel layout"):
            op.apply_forward_ewp(m)


def test_ewp_device_tensors_fp32_and_layout_refresh(btg):
    import torch

    blocks, m, d = R.random_problem(5, 6, 300, 40)
    spec = R.setup_full(blocks)
    with btg.setup(blocks, keep_channel_layout=True) as op:
        got = op.apply_forward_ewp(torch.from_numpy(m).cuda()).cpu().numpy()
        assert R.rel_l2(got, R.apply_forward(spec, m)) <= TOL64
        # F-hat rewritten by a new setup of the same rows: the layout is rebuilt
        blocks2, _, _ = R.random_problem(6, 6, 300, 40)
        op.setup_rows(blocks2, 0, 6)
        assert R.rel_l2(op.apply_adjoint_ewp(d), R.apply_adjoint(R.setup_full(blocks2), d)) <= TOL64
    with btg.setup(blocks, keep_channel_layout=True, precision=32) as op:
        assert R.rel_l2(op.apply_forward_ewp(m), R.apply_forward(spec, m)) <= 1e-5
