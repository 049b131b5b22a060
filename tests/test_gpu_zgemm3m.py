"""Multi-RHS Fourier step on DMMA with 3M complex products (csrc/btg_zgemm.cu,
the default): parity against the oracle on inputs spanning many binades, and
agreement with the 4M real-embedding kernels (BTG_ZGEMM_4M=1, read once per
process, so that arm runs in a subprocess). FP64 bar: relative L2 <= 1e-12."""

import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _problem(nd, nm, nt, nrhs, seed, wide):
    blocks, _, _ = R.random_problem(seed, nd, nm, nt)
    rng = np.random.default_rng(seed)
    M = rng.uniform(-1, 1, size=(nrhs, nm, nt))
    D = rng.uniform(-1, 1, size=(nrhs, nd, nt))
    if wide:
        blocks = blocks * np.exp2(rng.integers(-20, 4, size=blocks.shape))
        M = M * np.exp2(rng.integers(-12, 12, size=(nrhs, nm, 1)))
        D = D * np.exp2(rng.integers(-12, 12, size=(nrhs, nd, 1)))
    return blocks, M, D


@pytest.mark.parametrize("dims", [(130, 700, 16, 40), (16, 2000, 32, 3)])
def test_zgemm3m_wide_dynamic_range(dims):
    import paper_2407_13066_b200 as btg

    nd, nm, nt, nrhs = dims
    blocks, M, D = _problem(nd, nm, nt, nrhs, 4100 + nd, wide=True)
    spec = R.setup_full(blocks)
    with btg.setup(blocks) as op:
        F = op.apply_forward(M)
        A = op.apply_adjoint(D)
    for r in range(nrhs):
        assert R.rel_l2(F[r], R.apply_forward(spec, M[r])) <= TOL64
        assert R.rel_l2(A[r], R.apply_adjoint(spec, D[r])) <= TOL64


_ARM = """
import sys, numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import paper_2407_13066_b200 as btg
from test_gpu_zgemm3m import _problem
blocks, M, D = _problem(72, 1500, 24, 9, 4242, wide=False)
with btg.setup(blocks) as op:
    np.savez({out!r}, F=op.apply_forward(M), A=op.apply_adjoint(D))
"""


def test_zgemm3m_matches_4m(tmp_path):
    outs = {}
    for arm, env_extra in (("3m", {}), ("4m", {"BTG_ZGEMM_4M": "1"})):
        out = str(tmp_path / f"{arm}.npz")
        env = dict(os.environ, **env_extra)
        env.pop("BTG_ZGEMM_4M", None) if arm == "3m" else None
        code = _ARM.format(root=ROOT, tests=os.path.join(ROOT, "tests"), out=out)
        subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=300)
        outs[arm] = np.load(out)
    for k in ("F", "A"):
        a, b = outs["3m"][k], outs["4m"][k]
        assert a.shape == b.shape
        assert R.rel_l2(a, b) <= 1e-13
