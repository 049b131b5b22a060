"""Processor-grid planning over the native library (csrc/btg_planner.cu).

* :func:`plan_grid_b200` — the B200 / NVSwitch planner: the modelled time of
  the grid engine's own schedule (worst shard's HBM stream and vector
  transforms + NCCL ring collectives at NVLink-5 rates) for every
  factorisation of the worker count; returns the cheapest and the table.
* :func:`select_grid` — the reference's criterion (grid_planner.hpp:43-65):
  the scale-free cost (r/p) ln r + (10^l / r) ln(p/r), l = log10(N_d / N_m),
  minimised and snapped to a factorisation of p with the reference's
  preferences; checked against the reference build in tests/test_planner.py.
"""

from __future__ import annotations

import ctypes
import math
from typing import Tuple

from . import _lib
from ._lib import check

__all__ = ["select_grid", "weak_scaling_shape", "modified_cost", "comm_cost", "plan_grid", "parse_grid",
           "plan_grid_b200", "default_hw_model"]


def default_hw_model() -> dict:
    """The planner's default B200 rates (btg_default_hw_model)."""
    h = _lib.HwModel()
    check(_lib.load().btg_default_hw_model(ctypes.byref(h)))
    return {k: getattr(h, k) for k, _ in _lib.HwModel._fields_}


def plan_grid_b200(num_sensors: int, num_sources: int, num_steps: int, workers: int, action: str = "hessian",
                   precision: int = 64, hw: dict | None = None):
    """btg_plan_grid: ((rows, cols), table) where table rows are dicts with the
    modelled seconds (total, local, comm) of ``action`` on each r x c grid."""
    kinds = {"forward": _lib.BTG_GRID_FORWARD, "adjoint": _lib.BTG_GRID_ADJOINT, "hessian": _lib.BTG_GRID_HESSIAN}
    hm = None
    if hw is not None:
        base = default_hw_model()
        base.update(hw)
        hm = _lib.HwModel(**base)
    best = _lib.GridPlan()
    cnt = ctypes.c_size_t()
    args = (int(num_sensors), int(num_sources), int(num_steps), int(workers), int(precision), kinds[action],
            ctypes.byref(hm) if hm is not None else None)
    check(_lib.load().btg_plan_grid(*args, ctypes.byref(best), None, 0, ctypes.byref(cnt)))
    table = (_lib.GridPlan * max(1, cnt.value))()
    check(_lib.load().btg_plan_grid(*args, None, table, cnt.value, ctypes.byref(cnt)))
    rows = [{k: getattr(t, k) for k, _ in _lib.GridPlan._fields_} for t in table[:cnt.value]]
    return (int(best.rows), int(best.cols)), rows


def select_grid(workers: int, log_dim_ratio: float, gpus_per_node: int = 1) -> Tuple[int, int]:
    """select_grid (grid_planner.cpp:123-193)."""
    r, c = ctypes.c_size_t(), ctypes.c_size_t()
    check(_lib.load().btg_select_grid(int(workers), float(log_dim_ratio), int(gpus_per_node), ctypes.byref(r),
                                      ctypes.byref(c)))
    return int(r.value), int(c.value)


def weak_scaling_shape(local_ratio: float, workers: int) -> Tuple[bool, Tuple[int, int]]:
    """weak_scaling_shape (grid_planner.cpp:195-207): (indifferent, (rows, cols))."""
    ind, r, c = ctypes.c_int(), ctypes.c_size_t(), ctypes.c_size_t()
    check(_lib.load().btg_weak_scaling_shape(float(local_ratio), int(workers), ctypes.byref(ind), ctypes.byref(r),
                                             ctypes.byref(c)))
    return bool(ind.value), (int(r.value), int(c.value))


def modified_cost(rows: float, workers: int, log_dim_ratio: float) -> float:
    """modified_cost (grid_planner.cpp:116-121)."""
    v = ctypes.c_double()
    check(_lib.load().btg_modified_cost(float(rows), int(workers), float(log_dim_ratio), ctypes.byref(v)))
    return v.value


def comm_cost(grid: Tuple[int, int], num_sources: int, num_sensors: int, num_steps: int,
              latency: float = 1e-6, bandwidth: float = 1e10) -> float:
    """comm_cost (grid_planner.cpp:105-114), seconds per F + F* pair."""
    v = ctypes.c_double()
    check(_lib.load().btg_comm_cost(int(grid[0]), int(grid[1]), int(num_sources), int(num_sensors),
                                    int(num_steps), float(latency), float(bandwidth), ctypes.byref(v)))
    return v.value


def plan_grid(num_sensors: int, num_sources: int, workers: int, gpus_per_node: int = 1) -> Tuple[int, int]:
    """The grid for a global N_d x N_m operator on ``workers`` GPUs."""
    return select_grid(workers, math.log10(num_sensors / num_sources), gpus_per_node)


def parse_grid(text: str) -> Tuple[int, int]:
    """GridShape::parse (grid_planner.cpp:80-95): "RxC"."""
    pos = next((k for k, ch in enumerate(text) if ch in "xX"), -1)
    if pos <= 0 or pos + 1 >= len(text):
        raise _lib.Error(f"grid shape: expected RxC, got '{text}'")
    try:
        r, c = int(text[:pos]), int(text[pos + 1:])
    except ValueError:
        raise _lib.Error(f"grid shape: expected RxC, got '{text}'") from None
    if r <= 0 or c <= 0:
        raise _lib.Error("grid shape: rows and cols must be positive")
    return r, c


def conventional_cost_estimate(grid_points: float, num_steps: float, num_sensors: float,
                               rank_fraction: float = 0.1) -> dict:
    """conventional_cost_estimate (grid_planner.cpp:282-299), as the reference module's dict."""
    v = (ctypes.c_double * 7)()
    check(_lib.load().btg_conventional_cost_estimate(float(grid_points), float(num_steps), float(num_sensors),
                                                     float(rank_fraction), ctypes.byref(v)))
    keys = ("per_solve_flops", "effective_rank", "conventional_total_flops", "fft_setup_flops",
            "fft_matvec_flops", "fft_total_flops", "ratio")
    return dict(zip(keys, list(v)))


def apply_arithmetic_intensity(local_sensors: float, local_sources: float) -> float:
    """apply_arithmetic_intensity (grid_planner.cpp:301-304)."""
    return float(_lib.load().btg_apply_arithmetic_intensity(float(local_sensors), float(local_sources)))

