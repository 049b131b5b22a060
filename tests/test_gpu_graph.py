"""Device-pointer btg_hessian calls replay a captured CUDA graph of the whole
F -> C2R(Gamma^-1) -> R2C -> F* -> C2R(alpha R v) chain while the pointers and
epilogue match (inverse.cpp:78-91). The replay must give
the eager chain's bits (BTG_NO_GRAPH=1), follow new data in the same buffers,
re-capture on new pointers / parameters, and keep the counters' op model."""

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def btg():
    import paper_2407_13066_b200 as m

    return m


def _hess(btg, op, v, out, nrhs, gam, gkind, alpha, reg):
    from paper_2407_13066_b200 import _lib

    L = _lib.load()
    op._bind_stream(v)
    _lib.check(L.btg_hessian(op._h, v.data_ptr(), v.numel(), out.data_ptr(), out.numel(), nrhs,
                             gam.data_ptr() if gam is not None else None, gkind, float(alpha), reg,
                             _lib.BTG_DEVICE_PTRS))


@pytest.mark.parametrize("nrhs,precision", [(1, 64), (3, 64), (2, 32)])
def test_hessian_graph_replay_matches_eager(btg, monkeypatch, nrhs, precision):
    import torch

    blocks, _, _ = R.random_problem(91, 5, 40, 64)
    nt, nd, nm = blocks.shape
    rng = np.random.default_rng(5)
    gam = torch.from_numpy(rng.uniform(0.5, 2.0, nd)).cuda()
    with btg.setup(blocks, precision=precision) as op:
        v = torch.empty((nrhs * nm, nt), dtype=torch.float64, device="cuda")
        out = torch.empty_like(v)
        results = {}
        for mode in ("graph", "eager"):
            if mode == "eager":
                monkeypatch.setenv("BTG_NO_GRAPH", "1")
            else:
                monkeypatch.delenv("BTG_NO_GRAPH", raising=False)
            got = []
            op.reset_counters()
            for k, (alpha, reg, gk) in enumerate([(0.1, 1, 1), (0.1, 1, 1), (0.1, 1, 1), (0.0, 0, 0),
                                                   (0.25, 0, 1), (0.25, 0, 1)]):
                v.copy_(torch.from_numpy(np.random.default_rng(100 + k).uniform(-1, 1, (nrhs * nm, nt))))
                _hess(btg, op, v, out, nrhs, gam if gk else None, gk, alpha, reg)
                got.append(out.cpu().numpy().copy())
            results[mode] = (got, op.counters())
        monkeypatch.delenv("BTG_NO_GRAPH", raising=False)
    (gg, cg), (ge, ce) = results["graph"], results["eager"]
    for a, b in zip(gg, ge):
        assert np.array_equal(a, b)
    assert cg["launches"] == ce["launches"]
    assert cg["apply"]["bytes"] == ce["apply"]["bytes"]
    # and the chain is the Hessian: the last call against the oracle
    spec = R.setup_full(blocks)
    vlast = np.random.default_rng(105).uniform(-1, 1, (nrhs * nm, nt))
    for r in range(nrhs):
        want = R.gauss_newton_apply(spec, vlast[r * nm:(r + 1) * nm], gam.cpu().numpy(), 0.25, 0)
        tol = 1e-12 if precision == 64 else 1e-5
        assert R.rel_l2(gg[-1][r * nm:(r + 1) * nm], want) <= tol
