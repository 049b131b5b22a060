"""Inverse-problem caller of the Hessian action.

Mirrors ``btoep::cg_solve`` / ``objective_eval`` (``src/inverse.cpp:93-156``)
and the reference's Python ``cg_solve(blocks, d_obs, ...)`` binding
(``python/src/bindings.cpp:229-249``). The whole CG iteration runs in HBM
through ``btg_cg_solve``: Hessian actions, fused update / norm kernels and
deterministic dot products; only per-iteration scalars reach the host.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import BTG_DEVICE_PTRS, check
from .operator import _REG, SpectralOperator, _is_torch, setup

__all__ = ["cg_solve_op", "cg_solve", "objective_eval"]


def cg_solve_op(op: SpectralOperator, rhs, alpha: float = 1e-2, reg="identity", tol: float = 1e-8,
                maxiter: int = 0, precondition: bool = False, gamma_inv=None):
    """Solve (F* Gamma^-1 F + alpha R) m = rhs on the device. Returns
    (m, iterations, relative_residual, converged) like the reference binding."""
    reg_kind = _REG.get(reg)
    if reg_kind is None:
        raise _lib.Error(f"unknown regularization '{reg}' (expected identity or temporal-laplacian)")
    nrhs, _ = op._check_vec(rhs, op.num_sources, "cg_solve")
    if nrhs != 1:
        raise _lib.DimensionError("cg_solve: one right-hand side")
    on_dev = _is_torch(rhs)
    g_kind, g_ptr, g_keep = op._gamma(gamma_inv, on_dev)
    res = _lib.CgResult()
    L = _lib.load()
    if on_dev:
        import torch

        rhs = op._prep_torch(rhs)
        x = torch.empty_like(rhs)
        op._bind_stream(rhs)
        check(L.btg_cg_solve(op._h, rhs.data_ptr(), rhs.numel(), x.data_ptr(), x.numel(), g_ptr, g_kind,
                             float(alpha), reg_kind, float(tol), int(maxiter), int(precondition), BTG_DEVICE_PTRS,
                             ctypes.byref(res)))
    else:
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.empty_like(rhs)
        op._bind_stream(None)
        check(L.btg_cg_solve(op._h, rhs.ctypes.data, rhs.size, x.ctypes.data, x.size, g_ptr, g_kind, float(alpha),
                             reg_kind, float(tol), int(maxiter), int(precondition), 0, ctypes.byref(res)))
    del g_keep
    return x, int(res.iterations), float(res.relative_residual), bool(res.converged)


def cg_solve(blocks, d_obs, alpha: float = 1e-2, reg="identity", tol: float = 1e-8, maxiter: int = 0,
             precondition: bool = False, grid: str = "1x1", gamma_inv=None):
    """The reference binding's signature (bindings.cpp:229-249): setup from
    (steps, sensors, sources) blocks, rhs = F* d_obs, CG on the Hessian. With a
    grid other than 1x1 the right-hand side comes from distributed_adjoint on
    a single-process Partition of the blocks, as the reference does; the CG
    iterations run on the full device operator (the same H, so only the
    summation order of H v differs)."""
    from .distributed import Partition
    from .planner import parse_grid

    rows, cols = parse_grid(grid) if grid else (1, 1)
    op = blocks if isinstance(blocks, SpectralOperator) else setup(blocks)
    try:
        dw = d_obs if gamma_inv is None else _weighted(op, d_obs, gamma_inv)
        if (rows, cols) != (1, 1):
            with Partition(op if isinstance(blocks, SpectralOperator) else blocks, (rows, cols)) as p:
                rhs = p.adjoint(dw)
        else:
            rhs = op.apply_adjoint(dw)
        return cg_solve_op(op, rhs, alpha=alpha, reg=reg, tol=tol, maxiter=maxiter, precondition=precondition,
                           gamma_inv=gamma_inv)
    finally:
        if op is not blocks:
            op.close()


def _weighted(op, d, gamma_inv):
    g = np.asarray(gamma_inv, dtype=np.float64)
    return np.asarray(d) * (g[:, None] if g.ndim == 1 else g)


def objective_eval(op: SpectralOperator, m, d_obs, alpha: float = 0.0, reg="identity") -> float:
    """1/2 |F m - d_obs|^2 + alpha/2 m^T R m (inverse.cpp:93-103), on the device."""
    reg_kind = _REG.get(reg)
    if reg_kind is None:
        raise _lib.Error(f"unknown regularization '{reg}'")
    op._check_vec(m, op.num_sources, "objective")
    if tuple(d_obs.shape) != (op.num_sensors, op.num_steps):
        raise _lib.DimensionError("objective: observations do not match the operator")
    out = ctypes.c_double()
    L = _lib.load()
    if _is_torch(m):
        m, d_obs = op._prep_torch(m), op._prep_torch(d_obs)
        op._bind_stream(m)
        check(L.btg_objective(op._h, m.data_ptr(), m.numel(), d_obs.data_ptr(), d_obs.numel(), float(alpha),
                              reg_kind, BTG_DEVICE_PTRS, ctypes.byref(out)))
    else:
        m = np.ascontiguousarray(m, dtype=np.float64)
        d_obs = np.ascontiguousarray(d_obs, dtype=np.float64)
        op._bind_stream(None)
        check(L.btg_objective(op._h, m.ctypes.data, m.size, d_obs.ctypes.data, d_obs.size, float(alpha), reg_kind,
                              0, ctypes.byref(out)))
    return float(out.value)
