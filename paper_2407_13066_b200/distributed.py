"""2-D processor grid for the block-Toeplitz matvec over torch.distributed.

B200 form of the reference's distributed engine (``src/distributed.cpp``):
one process per GPU, rank ``i*cols + j`` owns grid cell (i, j) — the sensors
``[i*ceil(N_d/r), ...)`` x sources ``[j*ceil(N_m/c), ...)`` block of every
frequency (the ceiling partition, distributed.cpp:145-175) — and runs the
single-GPU pipeline (libbtg) on its shard. The reference's simulated
collectives become real NCCL collectives on row / column communicators:

* F  (distributed.cpp:312-351): column broadcast of the parameter slice from
  row 0, local F, row reduce (sum) onto column 0.
* F* (distributed.cpp:353-392): row broadcast of the data slice from column 0,
  local F*, column reduce onto row 0.
* Gauss-Newton Hessian (inverse.cpp:80-85 routed through a partition): the row
  reduce of F and the row broadcast of F* merge into one row all-reduce; Gamma^-1
  is applied in the local C2R epilogue (linear, so before the reduce) and
  alpha R v is added once, on row 0, in the final C2R epilogue.

The reductions are over time-domain d / m slices exactly as the reference does
them. Collective byte accounting mirrors the reference's CommLog
(distributed.hpp:77-92). With ``gloo`` and an injected host-side local
operator the same engine runs on CPU (tests/test_distributed.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

from ._lib import GridError

__all__ = ["Shard", "CommEvent", "partition_bounds", "GridEngine", "synthetic_shard_operator", "Partition",
           "partition_operator", "distributed_forward", "distributed_adjoint"]


@dataclass(frozen=True)
class Shard:
    """WorkerShard (distributed.hpp:27-40) without the operator payload."""

    grid_row: int
    grid_col: int
    sensor_begin: int
    sensor_end: int
    source_begin: int
    source_end: int

    @property
    def local_sensors(self) -> int:
        return self.sensor_end - self.sensor_begin

    @property
    def local_sources(self) -> int:
        return self.source_end - self.source_begin

    @property
    def empty(self) -> bool:
        return self.local_sensors == 0 or self.local_sources == 0


def partition_bounds(num_sensors: int, num_sources: int, rows: int, cols: int) -> List[Shard]:
    """partition_skeleton (distributed.cpp:145-175), row-major over the grid."""
    if rows <= 0 or cols <= 0:
        raise GridError("partition: grid must be positive")
    if rows > num_sensors or cols > num_sources:
        raise GridError(f"partition: grid {rows}x{cols} leaves workers without any of {num_sensors} sensors x "
                        f"{num_sources} sources")
    sc = -(-num_sensors // rows)
    mc = -(-num_sources // cols)
    return [Shard(i, j, min(i * sc, num_sensors), min((i + 1) * sc, num_sensors),
                  min(j * mc, num_sources), min((j + 1) * mc, num_sources))
            for i in range(rows) for j in range(cols)]


def _tree_depth(participants: int) -> int:
    depth, reach = 0, 1
    while reach < participants:
        reach *= 2
        depth += 1
    return depth


@dataclass
class CommEvent:
    """CommEvent (distributed.hpp:77-84)."""

    phase: str
    participants: int
    link_bytes: int
    messages: int = 0
    total_bytes: int = 0
    tree_depth: int = 0

    def __post_init__(self):
        self.messages = max(self.participants - 1, 0)
        self.total_bytes = self.messages * self.link_bytes
        self.tree_depth = _tree_depth(self.participants)


def synthetic_shard_operator(num_sensors: int, num_sources: int, num_steps: int, shard: Shard, seed: int,
                             device: int, precision: int = 64, slab_bytes: int = 2 << 30):
    """Build a shard's F-hat from the indexable synthetic first block column
    (entry (k, i, j) = uniform(seed ^ ((k*N_d + i)*N_m + j))), slab by slab
    on the device, so any grid reproduces the same global operator."""
    import torch

    from .operator import create, fill_uniform

    nd, nm = shard.local_sensors, shard.local_sources
    op = create(nd, nm, num_steps, precision, device)
    rows = max(1, min(nd, slab_bytes // max(1, 8 * num_steps * nm)))
    dev = f"cuda:{device}"
    for r0 in range(0, nd, rows):
        r1 = min(nd, r0 + rows)
        buf = torch.empty((num_steps, r1 - r0, nm), dtype=torch.float64, device=dev)
        offset = (shard.sensor_begin + r0) * num_sources + shard.source_begin
        fill_uniform(buf, seed, offset=offset, strides=(num_sensors * num_sources, num_sources))
        op.setup_rows(buf, r0, r1)
        del buf
    torch.cuda.synchronize(device)
    return op


class GridEngine:
    """F / F* / Hessian on an r x c grid of ranks (one GPU each).

    ``local_op`` is the shard's operator (a :class:`SpectralOperator`, or any
    object with the same ``apply_forward(x, gamma_inv=)`` /
    ``apply_adjoint(y, reg_v=, alpha=, reg=)`` methods on torch tensors); it
    is None for an empty shard. Vector slices are torch tensors on ``device``:
    parameter slices (local_sources x N_t) live on row-0 ranks, data slices
    (local_sensors x N_t) on column-0 ranks, as in the reference
    (scatter_param / scatter_data, distributed.hpp:66-73)."""

    def __init__(self, num_sensors: int, num_sources: int, num_steps: int, grid: Tuple[int, int], local_op,
                 device=None, process_group=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.torch = torch
        self.rows, self.cols = grid
        self.num_sensors, self.num_sources, self.num_steps = num_sensors, num_sources, num_steps
        self.world = dist.get_world_size(process_group)
        self.rank = dist.get_rank(process_group)
        if self.world != self.rows * self.cols:
            raise GridError(f"grid {self.rows}x{self.cols} needs {self.rows * self.cols} ranks, have {self.world}")
        self.shards = partition_bounds(num_sensors, num_sources, self.rows, self.cols)
        self.shard = self.shards[self.rank]
        self.local_op = local_op
        self.device = device if device is not None else torch.device("cpu")
        self.comm_log: List[CommEvent] = []
        # every rank creates every group, in the same order (torch.distributed rule)
        self._row_groups = [dist.new_group([i * self.cols + j for j in range(self.cols)]) for i in range(self.rows)]
        self._col_groups = [dist.new_group([i * self.cols + j for i in range(self.rows)]) for j in range(self.cols)]

    # -- construction helpers ---------------------------------------------------
    @classmethod
    def synthetic(cls, num_sensors: int, num_sources: int, num_steps: int, grid: Tuple[int, int], seed: int,
                  precision: int = 64):
        """Each rank builds its own shard of the synthetic operator on its GPU."""
        import torch
        import torch.distributed as dist

        rank = dist.get_rank()
        shard = partition_bounds(num_sensors, num_sources, *grid)[rank]
        device = torch.cuda.current_device()
        op = None if shard.empty else synthetic_shard_operator(num_sensors, num_sources, num_steps, shard, seed,
                                                               device, precision)
        return cls(num_sensors, num_sources, num_steps, grid, op, device=torch.device(f"cuda:{device}"))

    @classmethod
    def from_blocks(cls, blocks, grid: Tuple[int, int], precision: int = 64):
        """partition_operator (distributed.cpp:179-196): every rank transforms
        its rectangle of the host (steps, sensors, sources) first block column."""
        import numpy as np
        import torch
        import torch.distributed as dist

        from .operator import setup

        nt, nd, nm = blocks.shape
        shard = partition_bounds(nd, nm, *grid)[dist.get_rank()]
        device = torch.cuda.current_device()
        op = None
        if not shard.empty:
            local = np.ascontiguousarray(blocks[:, shard.sensor_begin:shard.sensor_end,
                                                shard.source_begin:shard.source_end])
            op = setup(local, precision=precision, device=device)
        return cls(nd, nm, nt, grid, op, device=torch.device(f"cuda:{device}"))

    @classmethod
    def from_file(cls, path, grid: Tuple[int, int], precision: int = 64):
        """Every rank loads only its rectangle of a reference operator file:
        time domain -> local setup; frequency domain -> the stored blocks of the
        rectangle, no re-setup (partition_operator(SpectralP2O),
        distributed.cpp:198-218)."""
        import torch
        import torch.distributed as dist

        from .io import load_operator_rect, peek_operator

        h = peek_operator(path)
        nd, nm, nt = int(h["num_sensors"]), int(h["num_sources"]), int(h["num_steps"])
        shard = partition_bounds(nd, nm, *grid)[dist.get_rank()]
        device = torch.cuda.current_device()
        op = None
        if not shard.empty:
            op = load_operator_rect(path, (shard.sensor_begin, shard.sensor_end),
                                    (shard.source_begin, shard.source_end), precision, device)
        return cls(nd, nm, nt, grid, op, device=torch.device(f"cuda:{device}"))

    @classmethod
    def from_operator(cls, op, grid: Tuple[int, int]):
        """partition_operator(const SpectralP2O&) (distributed.cpp:198-218) of an
        operator already resident on this rank's GPU (e.g. a replicated load):
        the rank keeps only its rectangle (btg_slice_operator, HBM->HBM)."""
        import torch
        import torch.distributed as dist

        nd, nm, nt = op.num_sensors, op.num_sources, op.num_steps
        shard = partition_bounds(nd, nm, *grid)[dist.get_rank()]
        device = torch.cuda.current_device()
        local = None
        if not shard.empty:
            local = op.slice((shard.sensor_begin, shard.sensor_end), (shard.source_begin, shard.source_end),
                             device)
        return cls(nd, nm, nt, grid, local, device=torch.device(f"cuda:{device}"))

    @staticmethod
    def plan(num_sensors: int, num_sources: int, workers: Optional[int] = None,
             gpus_per_node: int = 1) -> Tuple[int, int]:
        """The planner's grid (select_grid, grid_planner.cpp:123-193) for the
        world size (or ``workers``)."""
        from .planner import plan_grid

        if workers is None:
            import torch.distributed as dist

            workers = dist.get_world_size()
        return plan_grid(num_sensors, num_sources, workers, gpus_per_node)

    # -- helpers -------------------------------------------------------------------
    def _rank_of(self, i: int, j: int) -> int:
        return i * self.cols + j

    def _zeros(self, dim: int):
        return self.torch.zeros((dim, self.num_steps), dtype=self.torch.float64, device=self.device)

    def _record(self, phase: str, participants: int, dim: int):
        self.comm_log.append(CommEvent(phase, participants, 8 * self.num_steps * dim))

    def _bcast(self, buf, src_rank: int, group, participants: int):
        if participants > 1 and buf.numel():
            self.dist.broadcast(buf, src=src_rank, group=group)

    def _check_slice(self, x, dim: int, what: str):
        if x is None:
            raise ValueError(f"{what}: this rank owns a slice and must pass it")
        if tuple(x.shape) != (dim, self.num_steps):
            from ._lib import DimensionError

            raise DimensionError(f"{what}: slice is {tuple(x.shape)}, expected ({dim}, {self.num_steps})")
        return x.contiguous()

    def param_slice_bounds(self, j: int) -> Tuple[int, int]:
        s = self.shards[self._rank_of(0, j)]
        return s.source_begin, s.source_end

    def data_slice_bounds(self, i: int) -> Tuple[int, int]:
        s = self.shards[self._rank_of(i, 0)]
        return s.sensor_begin, s.sensor_end

    # -- the three actions ---------------------------------------------------------
    def forward(self, m_slice=None):
        """distributed_forward (distributed.cpp:312-351). Row-0 ranks pass their
        parameter slice; column-0 ranks get their data slice back (else None)."""
        sh, i, j = self.shard, self.shard.grid_row, self.shard.grid_col
        for jj in range(self.cols):
            s = self.shards[self._rank_of(0, jj)]
            self._record("broadcast", self.rows, s.local_sources)
        buf = self._check_slice(m_slice, sh.local_sources, "forward") if i == 0 else self._zeros(sh.local_sources)
        self._bcast(buf, self._rank_of(0, j), self._col_groups[j], self.rows)
        part = self.local_op.apply_forward(buf) if not sh.empty else self._zeros(sh.local_sensors)
        for ii in range(self.rows):
            self._record("reduce", self.cols, self.shards[self._rank_of(ii, 0)].local_sensors)
        if self.cols > 1 and part.numel():
            self.dist.reduce(part, dst=self._rank_of(i, 0), group=self._row_groups[i])
        return part if j == 0 else None

    def adjoint(self, d_slice=None):
        """distributed_adjoint (distributed.cpp:353-392). Column-0 ranks pass
        their data slice; row-0 ranks get their parameter slice back."""
        sh, i, j = self.shard, self.shard.grid_row, self.shard.grid_col
        for ii in range(self.rows):
            self._record("broadcast", self.cols, self.shards[self._rank_of(ii, 0)].local_sensors)
        buf = self._check_slice(d_slice, sh.local_sensors, "adjoint") if j == 0 else self._zeros(sh.local_sensors)
        self._bcast(buf, self._rank_of(i, 0), self._row_groups[i], self.cols)
        part = self.local_op.apply_adjoint(buf) if not sh.empty else self._zeros(sh.local_sources)
        for jj in range(self.cols):
            self._record("reduce", self.rows, self.shards[self._rank_of(0, jj)].local_sources)
        if self.rows > 1 and part.numel():
            self.dist.reduce(part, dst=self._rank_of(0, j), group=self._col_groups[j])
        return part if i == 0 else None

    def hessian(self, v_slice=None, alpha: float = 0.0, reg="identity", gamma_inv=None):
        """F* Gamma^-1 F v + alpha R v over the grid; row-0 ranks pass and receive
        parameter slices. gamma_inv is global ((N_d,) or (N_d, N_t)) on every rank."""
        sh, i, j = self.shard, self.shard.grid_row, self.shard.grid_col
        v = self._check_slice(v_slice, sh.local_sources, "hessian") if i == 0 else self._zeros(sh.local_sources)
        self._bcast(v, self._rank_of(0, j), self._col_groups[j], self.rows)
        g = None
        if gamma_inv is not None:
            g = gamma_inv[sh.sensor_begin:sh.sensor_end].contiguous()
        d = self.local_op.apply_forward(v, gamma_inv=g) if not sh.empty else self._zeros(sh.local_sensors)
        if self.cols > 1 and d.numel():
            self.dist.all_reduce(d, group=self._row_groups[i])  # reduce + broadcast of the reference, merged
        a = alpha if i == 0 else 0.0
        if not sh.empty:
            out = self.local_op.apply_adjoint(d, reg_v=v if a != 0.0 else None, alpha=a, reg=reg)
        else:
            out = self._zeros(sh.local_sources)
            if a != 0.0 and out.numel():
                raise GridError("hessian: an empty shard on row 0 cannot carry the regularization")
        if self.rows > 1 and out.numel():
            self.dist.reduce(out, dst=self._rank_of(0, j), group=self._col_groups[j])
        return out if i == 0 else None

    def comm_bytes(self) -> int:
        return sum(e.total_bytes for e in self.comm_log)

    def close(self):
        if self.local_op is not None and hasattr(self.local_op, "close"):
            self.local_op.close()
        self.local_op = None


# ---------------------------------------------------------------------------
# Single-process partition over the visible GPUs: the reference's Partition /
# distributed_forward / distributed_adjoint (distributed.hpp:43-121) and the
# module functions of the same names (python/src/bindings.cpp:148-172), over
# libbtg's btg_partition_* (one device handle per grid cell, placed round-robin
# on the device list; partial slices summed with the reference's fixed tree).
# ---------------------------------------------------------------------------
_BACKENDS = {"fft": 0, "ewp": 1, "naive": 2}


def _parse_backend(name: str) -> int:
    """parse_backend (distributed.cpp): "fft" | "ewp" | "naive"."""
    from ._lib import Error

    if name not in _BACKENDS:
        raise Error(f"unknown backend '{name}' (expected fft, ewp or naive)")
    return _BACKENDS[name]


class Partition:
    """partition_operator(CompactP2O | SpectralP2O, GridShape) (distributed.cpp:179-218)."""

    def __init__(self, source, grid, keep_channel_layout: bool = False, precision: int = 64, devices=None):
        import ctypes

        import numpy as np

        from . import _lib
        from .operator import SpectralOperator
        from .planner import parse_grid

        rows, cols = parse_grid(grid) if isinstance(grid, str) else (int(grid[0]), int(grid[1]))
        if devices is None:
            import torch

            devices = list(range(max(1, torch.cuda.device_count())))
        devs = (ctypes.c_int * len(devices))(*devices)
        h = ctypes.c_void_p()
        L = _lib.load()
        if isinstance(source, SpectralOperator):
            _lib.check(L.btg_partition_from_operator(source._h, rows, cols, devs, len(devices), ctypes.byref(h)))
            self.num_sensors, self.num_sources, self.num_steps = (source.num_sensors, source.num_sources,
                                                                  source.num_steps)
        else:
            b = np.ascontiguousarray(source, dtype=np.float64)
            if b.ndim != 3:
                raise _lib.DimensionError("blocks must be (steps, sensors, sources)")
            nt, nd, nm = b.shape
            flags = _lib.BTG_KEEP_CHANNEL_LAYOUT if keep_channel_layout else 0
            _lib.check(L.btg_partition_create(b.ctypes.data, nd, nm, nt, rows, cols, devs, len(devices),
                                              int(precision), flags, ctypes.byref(h)))
            self.num_sensors, self.num_sources, self.num_steps = nd, nm, nt
        self._h = h
        self.rows, self.cols = rows, cols

    def bounds(self):
        """(sensor_begin, sensor_end, source_begin, source_end) per shard, row-major."""
        import ctypes

        from . import _lib

        out = []
        for i in range(self.rows):
            for j in range(self.cols):
                b = (ctypes.c_size_t * 4)()
                _lib.check(_lib.load().btg_partition_shard(self._h, i, j, b, None))
                out.append(tuple(int(x) for x in b))
        return out

    def _apply(self, x, adjoint: bool, backend: str, parallel: bool):
        import numpy as np

        from . import _lib

        din, dout = (self.num_sensors, self.num_sources) if adjoint else (self.num_sources, self.num_sensors)
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (din, self.num_steps):
            raise _lib.DimensionError(f"distributed_{'adjoint' if adjoint else 'forward'}: vector is {x.shape}, "
                                      f"expected ({din}, {self.num_steps})")
        out = np.empty((dout, self.num_steps))
        fn = _lib.load().btg_partition_adjoint if adjoint else _lib.load().btg_partition_forward
        _lib.check(fn(self._h, x.ctypes.data, x.size, out.ctypes.data, out.size, _parse_backend(backend),
                      int(bool(parallel))))
        return out

    def forward(self, m, backend: str = "fft", parallel: bool = False):
        """distributed_forward (distributed.cpp:312-351)."""
        return self._apply(m, False, backend, parallel)

    def adjoint(self, d, backend: str = "fft", parallel: bool = False):
        """distributed_adjoint (distributed.cpp:353-392)."""
        return self._apply(d, True, backend, parallel)

    def close(self):
        if getattr(self, "_h", None):
            from . import _lib

            _lib.load().btg_partition_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def partition_operator(source, grid, keep_channel_layout: bool = False, precision: int = 64, devices=None):
    """partition_operator (distributed.hpp:57-66)."""
    return Partition(source, grid, keep_channel_layout, precision, devices)


def distributed_forward(blocks, m, grid: str = "1x1", backend: str = "fft", devices=None):
    """The reference module's distributed_forward(blocks, m, grid, backend)."""
    _parse_backend(backend)
    with Partition(blocks, grid, keep_channel_layout=backend == "ewp", devices=devices) as p:
        return p.forward(m, backend)


def distributed_adjoint(blocks, d, grid: str = "1x1", backend: str = "fft", devices=None):
    """The reference module's distributed_adjoint(blocks, d, grid, backend)."""
    _parse_backend(backend)
    with Partition(blocks, grid, keep_channel_layout=backend == "ewp", devices=devices) as p:
        return p.adjoint(d, backend)
