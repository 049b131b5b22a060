"""Processor-grid planner (grid_planner.hpp:43-65) over the native library.

``select_grid`` picks the r x c grid for p GPUs from l = log10(N_d / N_m): the
reference's scale-free cost (r/p) ln r + (10^l / r) ln(p/r) minimised and
snapped to a factorisation of p (exact integer minimiser for one GPU per node,
the node-divisibility preference when ``gpus_per_node`` > 1). On one NVSwitch
node every pair of B200s is one hop at full bandwidth, so this is an
orientation choice; :meth:`GridEngine.planned` uses it.
"""

from __future__ import annotations

import ctypes
import math
from typing import Tuple

from . import _lib
from ._lib import check

__all__ = ["select_grid", "weak_scaling_shape", "modified_cost", "comm_cost", "plan_grid", "parse_grid"]


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

