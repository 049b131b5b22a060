"""ctypes wrapper over ``oracle/_ref/libbtoep_ref.so`` — the reference's own
CPU implementation (unmodified ``/root/reference/proj/src`` sources + the FFT
shim, built by ``oracle/Makefile``).

TEST INFRASTRUCTURE ONLY: used by ``tests/``, ``tests/golden/make_golden.py``,
``__graft_entry__.smoke()`` and the CPU legs of ``bench.py``. Never imported by
the product package.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_ref" / "libbtoep_ref.so"

_lib = None
_c_double_p = ctypes.POINTER(ctypes.c_double)
_size_t = ctypes.c_size_t


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} not built (run `make -C oracle`)")
        L = ctypes.CDLL(str(LIB_PATH))
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_rng_uniform.argtypes = [ctypes.c_uint64, _size_t, ctypes.c_double, ctypes.c_double, _c_double_p]
        L.ref_rng_raw.argtypes = [ctypes.c_uint64, _size_t, ctypes.POINTER(ctypes.c_uint64)]
        L.ref_setup.argtypes = [_c_double_p, _size_t, _size_t, _size_t]
        L.ref_setup.restype = ctypes.c_void_p
        L.ref_destroy.argtypes = [ctypes.c_void_p]
        L.ref_setup_channel_layout.argtypes = [_c_double_p, _size_t, _size_t, _size_t]
        L.ref_setup_channel_layout.restype = ctypes.c_void_p
        for name in ("ref_forward_ewp", "ref_adjoint_ewp"):
            getattr(L, name).argtypes = [ctypes.c_void_p, _c_double_p, _c_double_p]
        L.ref_spectrum.argtypes = [ctypes.c_void_p, _c_double_p]
        for name in ("ref_forward", "ref_adjoint"):
            getattr(L, name).argtypes = [ctypes.c_void_p, _c_double_p, _c_double_p, _c_double_p]
        L.ref_hessian.argtypes = [ctypes.c_void_p, _c_double_p, _c_double_p, ctypes.c_double, ctypes.c_int]
        for name in ("ref_naive_forward", "ref_naive_adjoint"):
            getattr(L, name).argtypes = [_c_double_p, _size_t, _size_t, _size_t, _c_double_p, _c_double_p]
        L.ref_partition.argtypes = [_c_double_p, _size_t, _size_t, _size_t, _size_t, _size_t]
        L.ref_partition.restype = ctypes.c_void_p
        L.ref_partition_destroy.argtypes = [ctypes.c_void_p]
        L.ref_partition_bounds.argtypes = [ctypes.c_void_p, ctypes.POINTER(_size_t)]
        for name in ("ref_distributed_forward", "ref_distributed_adjoint"):
            getattr(L, name).argtypes = [ctypes.c_void_p, _c_double_p, _c_double_p, ctypes.c_int]
        L.ref_distributed_hessian.argtypes = [ctypes.c_void_p, _c_double_p, _c_double_p, ctypes.c_double,
                                              ctypes.c_int, ctypes.c_int]
        L.ref_verify.argtypes = [ctypes.c_uint64, ctypes.c_char_p, _size_t, ctypes.POINTER(ctypes.c_int)]
        L.ref_write_compact.argtypes = [ctypes.c_char_p, _c_double_p, _size_t, _size_t, _size_t]
        L.ref_save_spectral.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.ref_load_spectral.argtypes = [ctypes.c_char_p]
        L.ref_load_spectral.restype = ctypes.c_void_p
        L.ref_write_vector.argtypes = [ctypes.c_char_p, _c_double_p, _size_t, _size_t]
        L.ref_read_vector.argtypes = [ctypes.c_char_p, _c_double_p, _size_t]
        L.ref_cg_solve.argtypes = [ctypes.c_void_p, _c_double_p, _c_double_p, ctypes.c_double, ctypes.c_int,
                                   ctypes.c_double, _size_t, ctypes.c_int, _c_double_p]
        L.ref_objective.argtypes = [ctypes.c_void_p, _c_double_p, _c_double_p, ctypes.c_double, ctypes.c_int,
                                    _c_double_p]
        _sz_p = ctypes.POINTER(_size_t)
        L.ref_select_grid.argtypes = [_size_t, ctypes.c_double, ctypes.c_uint, _sz_p]
        L.ref_weak_scaling_shape.argtypes = [ctypes.c_double, _size_t, _sz_p]
        L.ref_modified_cost.argtypes = [ctypes.c_double, _size_t, ctypes.c_double, _c_double_p]
        L.ref_comm_cost.argtypes = [_size_t, _size_t, _size_t, _size_t, _size_t, ctypes.c_double,
                                    ctypes.c_double, _c_double_p]
        L.ref_partition_spectral.argtypes = [ctypes.c_void_p, _size_t, _size_t]
        L.ref_partition_spectral.restype = ctypes.c_void_p
        L.ref_partition_shard_spectrum.argtypes = [ctypes.c_void_p, _size_t, _size_t, _c_double_p]
        _lib = L
    return _lib


class RefError(ValueError):
    pass


def _check(rc):
    if rc != 0:
        raise RefError(lib().ref_last_error().decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(_c_double_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def rng_uniform(seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _check(lib().ref_rng_uniform(seed, n, lo, hi, _p(out)))
    return out


def rng_raw(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    _check(lib().ref_rng_raw(seed, n, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return out


class RefSpectralOperator:
    """btoep::SpectralP2O built by the reference's setup (block_operator.cpp:178-205)."""

    def __init__(self, blocks: np.ndarray, keep_channel_layout: bool = False):
        self.blocks = _f64(blocks)
        nt, nd, nm = self.blocks.shape
        self.num_steps, self.num_sensors, self.num_sources = nt, nd, nm
        setup = lib().ref_setup_channel_layout if keep_channel_layout else lib().ref_setup
        h = setup(_p(self.blocks), nd, nm, nt)
        if not h:
            raise RefError(lib().ref_last_error().decode())
        self._h = ctypes.c_void_p(h)

    def close(self):
        if self._h:
            lib().ref_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def freq_blocks(self) -> np.ndarray:
        out = np.empty((2 * self.num_steps, self.num_sensors, self.num_sources), dtype=np.complex128)
        _check(lib().ref_spectrum(self._h, out.ctypes.data_as(_c_double_p)))
        return out

    def apply_forward(self, m, stage_seconds: np.ndarray | None = None) -> np.ndarray:
        m = _f64(m)
        d = np.empty((self.num_sensors, self.num_steps))
        _check(lib().ref_forward(self._h, _p(m), _p(d), None if stage_seconds is None else _p(stage_seconds)))
        return d

    def apply_adjoint(self, d, stage_seconds: np.ndarray | None = None) -> np.ndarray:
        d = _f64(d)
        m = np.empty((self.num_sources, self.num_steps))
        _check(lib().ref_adjoint(self._h, _p(d), _p(m), None if stage_seconds is None else _p(stage_seconds)))
        return m

    def apply_forward_ewp(self, m) -> np.ndarray:
        """apply_forward_ewp (block_operator.cpp:345-382); needs keep_channel_layout."""
        m = _f64(m)
        d = np.empty((self.num_sensors, self.num_steps))
        _check(lib().ref_forward_ewp(self._h, _p(m), _p(d)))
        return d

    def apply_adjoint_ewp(self, d) -> np.ndarray:
        """apply_adjoint_ewp (block_operator.cpp:384-421)."""
        d = _f64(d)
        m = np.empty((self.num_sources, self.num_steps))
        _check(lib().ref_adjoint_ewp(self._h, _p(d), _p(m)))
        return m

    def hessian_apply(self, v, alpha: float = 0.0, reg_kind: int = 0) -> np.ndarray:
        v = _f64(v)
        hv = np.empty_like(v)
        _check(lib().ref_hessian(self._h, _p(v), _p(hv), float(alpha), int(reg_kind)))
        return hv

    def cg_solve(self, rhs, alpha: float, reg_kind: int = 0, tol: float = 1e-8, maxiter: int = 0,
                 precondition: bool = False):
        """btoep::cg_solve (inverse.cpp:105-156): (x, iterations, relative_residual, converged)."""
        rhs = _f64(rhs)
        x = np.empty_like(rhs)
        out = np.zeros(3)
        _check(lib().ref_cg_solve(self._h, _p(rhs), _p(x), float(alpha), int(reg_kind), float(tol), int(maxiter),
                                  int(precondition), _p(out)))
        return x, int(out[0]), float(out[1]), bool(out[2])

    def objective(self, m, d_obs, alpha: float, reg_kind: int = 0) -> float:
        v = np.zeros(1)
        _check(lib().ref_objective(self._h, _p(_f64(m)), _p(_f64(d_obs)), float(alpha), int(reg_kind), _p(v)))
        return float(v[0])


def write_compact(path, blocks) -> None:
    """io::write_operator(CompactP2O) (io.cpp:97-111)."""
    blocks = _f64(blocks)
    nt, nd, nm = blocks.shape
    _check(lib().ref_write_compact(str(path).encode(), _p(blocks), nd, nm, nt))


def save_spectral(op: "RefSpectralOperator", path) -> None:
    """io::write_operator(SpectralP2O) (io.cpp:113-130)."""
    _check(lib().ref_save_spectral(op._h, str(path).encode()))


def load_spectral_spectrum(path, nd, nm, nt) -> np.ndarray:
    """io::read_spectral_operator (io.cpp:179-205) -> its freq_blocks."""
    h = lib().ref_load_spectral(str(path).encode())
    if not h:
        raise RefError(lib().ref_last_error().decode())
    out = np.empty((2 * nt, nd, nm), dtype=np.complex128)
    try:
        _check(lib().ref_spectrum(ctypes.c_void_p(h), out.ctypes.data_as(_c_double_p)))
    finally:
        lib().ref_destroy(ctypes.c_void_p(h))
    return out


def write_vector(path, v) -> None:
    v = _f64(v)
    _check(lib().ref_write_vector(str(path).encode(), _p(v), v.shape[0], v.shape[1]))


def read_vector(path, shape) -> np.ndarray:
    out = np.empty(shape)
    _check(lib().ref_read_vector(str(path).encode(), _p(out), out.size))
    return out


def naive_forward(blocks, m) -> np.ndarray:
    blocks, m = _f64(blocks), _f64(m)
    nt, nd, nm = blocks.shape
    d = np.empty((nd, nt))
    _check(lib().ref_naive_forward(_p(blocks), nd, nm, nt, _p(m), _p(d)))
    return d


def naive_adjoint(blocks, d) -> np.ndarray:
    blocks, d = _f64(blocks), _f64(d)
    nt, nd, nm = blocks.shape
    m = np.empty((nm, nt))
    _check(lib().ref_naive_adjoint(_p(blocks), nd, nm, nt, _p(d), _p(m)))
    return m


class RefPartition:
    """btoep::Partition (distributed.cpp:179-196) and its F / F* engine."""

    def __init__(self, blocks, rows: int, cols: int):
        self.blocks = _f64(blocks)
        nt, nd, nm = self.blocks.shape
        self.num_steps, self.num_sensors, self.num_sources = nt, nd, nm
        self.rows, self.cols = rows, cols
        h = lib().ref_partition(_p(self.blocks), nd, nm, nt, rows, cols)
        if not h:
            raise RefError(lib().ref_last_error().decode())
        self._h = ctypes.c_void_p(h)

    def __del__(self):
        try:
            if self._h:
                lib().ref_partition_destroy(self._h)
        except Exception:
            pass

    def bounds(self):
        out = (_size_t * (4 * self.rows * self.cols))()
        _check(lib().ref_partition_bounds(self._h, out))
        return [tuple(out[4 * w : 4 * w + 4]) for w in range(self.rows * self.cols)]

    def forward(self, m, parallel: bool = False) -> np.ndarray:
        m = _f64(m)
        d = np.empty((self.num_sensors, self.num_steps))
        _check(lib().ref_distributed_forward(self._h, _p(m), _p(d), int(parallel)))
        return d

    def adjoint(self, d, parallel: bool = False) -> np.ndarray:
        d = _f64(d)
        m = np.empty((self.num_sources, self.num_steps))
        _check(lib().ref_distributed_adjoint(self._h, _p(d), _p(m), int(parallel)))
        return m

    def hessian(self, v, alpha: float = 0.0, reg_kind: int = 0, parallel: bool = False) -> np.ndarray:
        v = _f64(v)
        hv = np.empty_like(v)
        _check(lib().ref_distributed_hessian(self._h, _p(v), _p(hv), float(alpha), int(reg_kind), int(parallel)))
        return hv


def verify(seed: int = 20240901):
    buf = ctypes.create_string_buffer(1 << 16)
    passed = ctypes.c_int(0)
    _check(lib().ref_verify(seed, buf, len(buf), ctypes.byref(passed)))
    return bool(passed.value), buf.value.decode()


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---- grid planner (grid_planner.hpp:43-65) ----------------------------------------
def select_grid(workers: int, log_dim_ratio: float, gpus_per_node: int = 1):
    rc = (_size_t * 2)()
    _check(lib().ref_select_grid(workers, log_dim_ratio, gpus_per_node, rc))
    return int(rc[0]), int(rc[1])


def weak_scaling_shape(local_ratio: float, workers: int):
    out = (_size_t * 3)()
    _check(lib().ref_weak_scaling_shape(local_ratio, workers, out))
    return bool(out[0]), (int(out[1]), int(out[2]))


def modified_cost(rows: float, workers: int, log_dim_ratio: float) -> float:
    v = ctypes.c_double()
    _check(lib().ref_modified_cost(rows, workers, log_dim_ratio, ctypes.byref(v)))
    return v.value


def comm_cost(rows, cols, num_sources, num_sensors, num_steps, latency=1e-6, bandwidth=1e10) -> float:
    v = ctypes.c_double()
    _check(lib().ref_comm_cost(rows, cols, num_sources, num_sensors, num_steps, latency, bandwidth,
                               ctypes.byref(v)))
    return v.value


def spectral_partition_shards(op: "RefSpectralOperator", rows: int, cols: int):
    """partition_operator(const SpectralP2O&) (distributed.cpp:198-218): the full
    2N_t frequency blocks of every shard, keyed by (row, col)."""
    L = lib()
    h = L.ref_partition_spectral(op._h, rows, cols)
    if not h:
        raise RefError(L.ref_last_error().decode())
    try:
        b = (_size_t * (4 * rows * cols))()
        _check(L.ref_partition_bounds(h, b))
        out = {}
        for k in range(rows * cols):
            r, c = divmod(k, cols)
            s0, s1, m0, m1 = (int(x) for x in b[4 * k: 4 * k + 4])
            if s1 == s0 or m1 == m0:
                continue
            spec = np.empty((2 * op.num_steps, s1 - s0, m1 - m0), dtype=np.complex128)
            _check(L.ref_partition_shard_spectrum(h, r, c, spec.ctypes.data_as(_c_double_p)))
            out[(r, c)] = (s0, s1, m0, m1, spec)
        return out
    finally:
        L.ref_partition_destroy(h)
