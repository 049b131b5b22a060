"""CPU restatement of the reference's block-Toeplitz matvec path.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module, and only as the checker. The product (``paper_2407_13066_b200``) never
imports it and has no CPU fallback.

Every function follows a reference routine (paths relative to
``/root/reference/proj``) in numpy float64/complex128. Parity of this
restatement is pinned two ways (see ``tests/test_oracle.py``): against the
golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by running the reference itself (``oracle/_ref/libbtoep_ref.so``,
built from the unmodified reference sources with only the FFTW wrapper
replaced), and against the reference's own known-answer tests (identity and
shift operators, 1x1 spectrum, conjugate symmetry, causality).
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "Mt19937_64",
    "ref_uniform",
    "random_problem",
    "setup_full",
    "apply_forward",
    "apply_adjoint",
    "hessian_apply",
    "gauss_newton_apply",
    "reg_apply",
    "naive_apply_forward",
    "naive_apply_adjoint",
    "dense_block_operator_soti",
    "rel_max_diff",
    "rel_l2",
    "partition_bounds",
    "tree_reduce",
]

# ---------------------------------------------------------------------------
# RNG: include/btoep/rng.hpp:12-32 (std::mt19937_64 + hand-rolled 53-bit
# uniform). Vectorized numpy restatement of the standard MT19937-64.
# ---------------------------------------------------------------------------
_MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)


class Mt19937_64:
    """std::mt19937_64 (rng.hpp:14) with numpy-vectorized twists."""

    n, m = 312, 156
    _A = np.uint64(0xB5026F5AA96619E9)
    _UPPER = np.uint64(0xFFFFFFFF80000000)
    _LOWER = np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [0] * self.n
        mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, self.n):
            prev = mt[i - 1]
            mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.mt = np.array(mt, dtype=np.uint64)
        self.idx = self.n

    def _twist(self):
        mt, n, m = self.mt, self.n, self.m
        up, lo, a = self._UPPER, self._LOWER, self._A

        def step(i0, i1, nxt, far):
            x = (mt[i0:i1] & up) | (nxt & lo)
            xa = x >> np.uint64(1)
            xa = np.where((x & np.uint64(1)) != 0, xa ^ a, xa)
            mt[i0:i1] = far ^ xa

        step(0, n - m, mt[1 : n - m + 1].copy(), mt[m:n].copy())
        step(n - m, n - 1, mt[n - m + 1 : n].copy(), mt[0 : m - 1].copy())
        step(n - 1, n, mt[0:1].copy(), mt[m - 1 : m].copy())
        self.idx = 0

    def next_u64(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        pos = 0
        while pos < count:
            if self.idx >= self.n:
                self._twist()
            take = min(count - pos, self.n - self.idx)
            y = self.mt[self.idx : self.idx + take].copy()
            y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
            y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
            y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
            y ^= y >> np.uint64(43)
            out[pos : pos + take] = y
            pos += take
            self.idx += take
        return out

    def uniform(self, count: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        """Rng::uniform(lo, hi) = lo + (hi - lo) * ((gen() >> 11) * 2^-53) (rng.hpp:16-18)."""
        u = (self.next_u64(count) >> np.uint64(11)).astype(np.float64) * (2.0**-53)
        return lo + (hi - lo) * u


def ref_uniform(seed: int, count: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    return Mt19937_64(seed).uniform(count, lo, hi)


def random_problem(seed: int, nd: int, nm: int, nt: int):
    """tests/oracles.cpp:87-98 draw order on one Rng: random_operator (blocks,
    TOSI (nt, nd, nm)), then random_vector m (nm x nt SOTI), then d (nd x nt)."""
    rng = Mt19937_64(seed)
    blocks = rng.uniform(nt * nd * nm, -1.0, 1.0).reshape(nt, nd, nm)
    m = rng.uniform(nm * nt, -1.0, 1.0).reshape(nm, nt)
    d = rng.uniform(nd * nt, -1.0, 1.0).reshape(nd, nt)
    return blocks, m, d


# ---------------------------------------------------------------------------
# FFT pipeline: src/block_operator.cpp. Full 2*N_t spectrum as the reference
# keeps it (block_operator.hpp:47).
# ---------------------------------------------------------------------------
def setup_full(blocks: np.ndarray) -> np.ndarray:
    """setup (block_operator.cpp:178-205): zero-pad each (sensor, source) series
    to 2*N_t, forward DFT (fft.cpp:38-40, unnormalized, sign -1), freq-major
    (2*N_t, N_d, N_m)."""
    blocks = np.asarray(blocks, dtype=np.float64)
    nt = blocks.shape[0]
    return np.fft.fft(blocks, n=2 * nt, axis=0)


def _pad_and_transform(v: np.ndarray) -> np.ndarray:
    """pad_and_transform (block_operator.cpp:54-80) followed by reorder_in
    (:231-236): returns freq-major (2*N_t, channels)."""
    nt = v.shape[1]
    return np.fft.fft(v, n=2 * nt, axis=1).T


def _transform_back_and_unpad(freq_major: np.ndarray, nt: int) -> np.ndarray:
    """reorder_out (:264-266) + transform_back_and_unpad (:83-121): inverse DFT
    scaled by 1/(2 N_t) (fft.cpp:42-46), keep t < N_t, real part."""
    return np.fft.ifft(freq_major.T, axis=1)[:, :nt].real.copy()


def apply_forward(spec: np.ndarray, m: np.ndarray) -> np.ndarray:
    """apply_forward (block_operator.cpp:218-273): d_f = F_f m_f per frequency,
    row dot products over j (:243-253)."""
    nt = m.shape[1]
    mh = _pad_and_transform(np.asarray(m, dtype=np.float64))
    dh = np.einsum("fij,fj->fi", spec, mh)
    return _transform_back_and_unpad(dh, nt)


def apply_adjoint(spec: np.ndarray, d: np.ndarray) -> np.ndarray:
    """apply_adjoint (block_operator.cpp:275-331): m_f = F_f^H d_f (:302-311)."""
    nt = d.shape[1]
    dh = _pad_and_transform(np.asarray(d, dtype=np.float64))
    mh = np.einsum("fij,fi->fj", np.conj(spec), dh)
    return _transform_back_and_unpad(mh, nt)


def reg_apply(v: np.ndarray, kind: int) -> np.ndarray:
    """Regularization::apply (inverse.cpp:32-49): kind 0 = identity, 1 = the
    clamped temporal Laplacian (2, -1 tridiagonal per source)."""
    v = np.asarray(v, dtype=np.float64)
    if kind == 0:
        return v.copy()
    out = 2.0 * v
    out[:, 1:] -= v[:, :-1]
    out[:, :-1] -= v[:, 1:]
    return out


def hessian_apply(spec, v, alpha=0.0, reg_kind=0):
    """HessianOperator::apply (inverse.cpp:78-91): F^T F v + alpha R v."""
    return apply_adjoint(spec, apply_forward(spec, v)) + alpha * reg_apply(v, reg_kind)


def gauss_newton_apply(spec, v, gamma_inv=None, alpha=0.0, reg_kind=0):
    """North-star Gauss-Newton action F* Gamma^-1 F v + alpha R v, composed from
    the reference's F and F* (no reference routine carries Gamma^-1; SURVEY
    §8c pins it by composition). gamma_inv: None, (N_d,) or (N_d, N_t)."""
    d = apply_forward(spec, v)
    if gamma_inv is not None:
        g = np.asarray(gamma_inv, dtype=np.float64)
        d = d * (g[:, None] if g.ndim == 1 else g)
    return apply_adjoint(spec, d) + alpha * reg_apply(v, reg_kind)


# ---------------------------------------------------------------------------
# Time-domain oracles: block_operator.cpp:423-482 and tests/oracles.cpp:42-69.
# ---------------------------------------------------------------------------
def naive_apply_forward(blocks, m):
    """naive_apply_forward (block_operator.cpp:423-452), SOTI in/out."""
    nt, nd, _ = blocks.shape
    d = np.zeros((nd, nt))
    for t_out in range(nt):
        for t_in in range(t_out + 1):
            d[:, t_out] += blocks[t_out - t_in] @ m[:, t_in]
    return d


def naive_apply_adjoint(blocks, d):
    """naive_apply_adjoint (block_operator.cpp:454-482), SOTI in/out."""
    nt, _, nm = blocks.shape
    m = np.zeros((nm, nt))
    for t_out in range(nt):
        for t_in in range(t_out + 1):
            m[:, t_in] += blocks[t_out - t_in].T @ d[:, t_out]
    return m


def dense_block_operator_soti(blocks):
    """dense_block_operator (tests/oracles.cpp:42-53) permuted to SOTI rows/cols
    (tests/test_inverse.cpp:17-30): (N_d N_t) x (N_m N_t)."""
    nt, nd, nm = blocks.shape
    mat = np.zeros((nd, nt, nm, nt))
    for bi in range(nt):
        for bj in range(bi + 1):
            mat[:, bi, :, bj] = blocks[bi - bj]
    return mat.reshape(nd * nt, nm * nt)


def rel_max_diff(a, b) -> float:
    """tests/oracles.cpp:71-79."""
    dt = np.complex128 if np.iscomplexobj(a) or np.iscomplexobj(b) else np.float64
    a = np.asarray(a, dtype=dt).ravel()
    b = np.asarray(b, dtype=dt).ravel()
    diff = np.max(np.abs(a - b)) if a.size else 0.0
    scale = max(np.max(np.abs(a)) if a.size else 0.0, np.max(np.abs(b)) if b.size else 0.0)
    return float(diff if scale == 0.0 else diff / scale)


def rel_l2(got, want) -> float:
    """North-star parity metric: ||got - want||_2 / ||want||_2."""
    dt = np.complex128 if np.iscomplexobj(got) or np.iscomplexobj(want) else np.float64
    got = np.asarray(got, dtype=dt).ravel()
    want = np.asarray(want, dtype=dt).ravel()
    den = np.linalg.norm(want)
    num = np.linalg.norm(got - want)
    return float(num if den == 0.0 else num / den)


# ---------------------------------------------------------------------------
# Distribution: src/distributed.cpp.
# ---------------------------------------------------------------------------
def partition_bounds(nd, nm, rows, cols):
    """partition_skeleton (distributed.cpp:145-175): ceiling chunks, trailing
    shards may be smaller or empty; rejects rows > N_d or cols > N_m.
    Returns a row-major list of (sensor_begin, sensor_end, source_begin, source_end)."""
    if rows == 0 or cols == 0:
        raise ValueError("partition: grid must be positive")
    if rows > nd or cols > nm:
        raise ValueError(f"partition: grid {rows}x{cols} leaves workers without any of "
                         f"{nd} sensors x {nm} sources")
    sc = -(-nd // rows)
    mc = -(-nm // cols)
    out = []
    for i in range(rows):
        for j in range(cols):
            out.append((min(i * sc, nd), min((i + 1) * sc, nd), min(j * mc, nm), min((j + 1) * mc, nm)))
    return out


def tree_reduce(partials):
    """tree_reduce (distributed.cpp:38-47): ((v0+v1)+(v2+v3))+... in place."""
    parts = [np.array(p, dtype=np.float64, copy=True) for p in partials]
    step = 1
    while step < len(parts):
        for i in range(0, len(parts) - step, 2 * step):
            parts[i] += parts[i + step]
        step *= 2
    return parts[0]


# ---------------------------------------------------------------------------
# Host twin of the product's indexable synthetic generator (btg_fill_uniform):
# value at global index g = lo + (hi-lo) * ((splitmix64(seed ^ g) >> 11) * 2^-53).
# Lets tests regenerate any slice of a device-generated full-size operator.
# ---------------------------------------------------------------------------
def splitmix_uniform(seed: int, idx, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ np.asarray(idx, dtype=np.uint64)
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return lo + (hi - lo) * ((z >> np.uint64(11)).astype(np.float64) * 2.0**-53)


def synthetic_blocks_slice(seed, nd, nm, nt, sensors, sources):
    """Entries (k, i, j) of the synthetic first block column for the given
    sensor / source index arrays: uniform(seed ^ ((k*N_d + i)*N_m + j))."""
    k = np.arange(nt, dtype=np.uint64)[:, None, None]
    i = np.asarray(sensors, dtype=np.uint64)[None, :, None]
    j = np.asarray(sources, dtype=np.uint64)[None, None, :]
    return splitmix_uniform(seed, (k * np.uint64(nd) + i) * np.uint64(nm) + j)
