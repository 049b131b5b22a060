"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

The reference CPU implementation is oracle/_ref/libbtoep_ref.so, built by
oracle/Makefile from the unmodified /root/reference/proj/src sources (only the
FFTW wrapper replaced). Inputs are the reference's own seeded streams
(tests/oracles.cpp:87-98: random_operator, then random_vector m, then d, all on
one btoep::Rng), so every fixture can be regenerated from its seed; the
fixtures store the seeds, a fingerprint of the inputs (to pin the RNG port) and
the reference's outputs.

    python tests/golden/make_golden.py      # (re)writes tests/golden/*.npz
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import refcpu  # noqa: E402
from oracle.restate import Mt19937_64  # noqa: E402

OUT = Path(__file__).resolve().parent


def ref_problem(seed, nd, nm, nt):
    """Same draw order as tests/oracles.cpp:87-98, drawn by the reference's Rng."""
    n = nt * nd * nm + nm * nt + nd * nt
    u = refcpu.rng_uniform(seed, n, -1.0, 1.0)
    blocks = u[: nt * nd * nm].reshape(nt, nd, nm)
    m = u[nt * nd * nm : nt * nd * nm + nm * nt].reshape(nm, nt)
    d = u[nt * nd * nm + nm * nt :].reshape(nd, nt)
    return blocks, m, d


def fingerprint(*arrays):
    return np.array([float(np.sum(a)) for a in arrays] + [float(a.ravel()[-1]) for a in arrays])


def config_a(seed, full):
    """configs[0]: N_t=64, N_d=8, N_m=256 (BASELINE.json)."""
    nd, nm, nt = 8, 256, 64
    blocks, m, d = ref_problem(seed, nd, nm, nt)
    op = refcpu.RefSpectralOperator(blocks)
    out = dict(seed=seed, dims=np.array([nd, nm, nt]), fingerprint=fingerprint(blocks, m, d),
               fwd=op.apply_forward(m), adj=op.apply_adjoint(d))
    if full:
        out["hess_a0"] = op.hessian_apply(m, 0.0, 0)
        out["hess_lap"] = op.hessian_apply(m, 0.1, 1)
        out["hess_id"] = op.hessian_apply(m, 0.25, 0)
        out["naive_fwd"] = refcpu.naive_forward(blocks, m)
        # F* Gamma^-1 F composed through the reference's own F and F*
        gamma = refcpu.rng_uniform(seed + 1, nd, 0.5, 2.0)
        out["gamma"] = gamma
        out["gn_gamma"] = op.apply_adjoint(gamma[:, None] * op.apply_forward(m))
    return out


def small_case():
    """test_block_operator.cpp:117-124 shape (3 sensors, 5 sources, 16 steps,
    seed 35) with its full reference spectrum."""
    blocks, m, d = ref_problem(35, 3, 5, 16)
    op = refcpu.RefSpectralOperator(blocks)
    return dict(blocks=blocks, m=m, d=d, spectrum=op.freq_blocks, fwd=op.apply_forward(m),
                adj=op.apply_adjoint(d), hess=op.hessian_apply(m, 0.1, 0))


def random_instances():
    """The 40 trials of test_block_operator.cpp:183-203 (Rng(43): sensors, sources,
    steps = 1 + integer(8|8|48), then operator, m, d), with the reference's FFT
    and naive results. Ragged and non-power-of-two lengths, including primes."""
    rng = Mt19937_64(43)
    dims, fwd, adj, nf, na = [], [], [], [], []
    for _ in range(40):
        sensors = 1 + int(rng.next_u64(1)[0] % np.uint64(8))
        sources = 1 + int(rng.next_u64(1)[0] % np.uint64(8))
        steps = 1 + int(rng.next_u64(1)[0] % np.uint64(48))
        blocks = rng.uniform(steps * sensors * sources, -1.0, 1.0).reshape(steps, sensors, sources)
        m = rng.uniform(sources * steps, -1.0, 1.0).reshape(sources, steps)
        d = rng.uniform(sensors * steps, -1.0, 1.0).reshape(sensors, steps)
        op = refcpu.RefSpectralOperator(blocks)
        dims.append((sensors, sources, steps))
        fwd.append(op.apply_forward(m).ravel())
        adj.append(op.apply_adjoint(d).ravel())
        nf.append(refcpu.naive_forward(blocks, m).ravel())
        na.append(refcpu.naive_adjoint(blocks, d).ravel())
    cat = lambda xs: np.concatenate(xs)  # noqa: E731
    return dict(dims=np.array(dims), fwd=cat(fwd), adj=cat(adj), naive_fwd=cat(nf), naive_adj=cat(na))


def distributed_case():
    """test_smoke.py:68-78 grids on a (5 sensors, 7 sources, 12 steps) problem."""
    blocks, m, d = ref_problem(5, 5, 7, 12)
    out = {}
    for grid in ("1x4", "2x2", "4x1", "2x3"):
        r, c = map(int, grid.split("x"))
        part = refcpu.RefPartition(blocks, r, c)
        out[f"fwd_{grid}"] = part.forward(m)
        out[f"adj_{grid}"] = part.adjoint(d)
        out[f"bounds_{grid}"] = np.array(part.bounds())
    return out


def ewp_case():
    """EWP backend (apply_forward_ewp / apply_adjoint_ewp, block_operator.cpp:345-421)
    on a reference operator set up with keep_channel_layout: configs[0] with seed
    1 and a ragged 7 x 45 x 37 case."""
    out = {}
    for tag, (seed, nd, nm, nt) in (("a", (1, 8, 256, 64)), ("r", (77, 7, 45, 37))):
        blocks, m, d = ref_problem(seed, nd, nm, nt)
        op = refcpu.RefSpectralOperator(blocks, keep_channel_layout=True)
        out[f"{tag}_seed"] = seed
        out[f"{tag}_dims"] = np.array([nd, nm, nt])
        out[f"{tag}_fingerprint"] = fingerprint(blocks, m, d)
        out[f"{tag}_fwd"] = op.apply_forward_ewp(m)
        out[f"{tag}_adj"] = op.apply_adjoint_ewp(d)
    return out


def main():
    np.savez_compressed(OUT / "ewp_case.npz", **ewp_case())
    np.savez_compressed(OUT / "config_a_seed1.npz", **config_a(1, full=True))
    np.savez_compressed(OUT / "config_a_seed20240901.npz", **config_a(20240901, full=False))
    np.savez_compressed(OUT / "small_case.npz", **small_case())
    np.savez_compressed(OUT / "random_instances.npz", **random_instances())
    np.savez_compressed(OUT / "distributed_case.npz", **distributed_case())
    ok, report = refcpu.verify(20240901)
    (OUT / "reference_verify.txt").write_text(report)
    assert ok, report
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
