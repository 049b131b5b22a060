"""2-D processor grid for the block-Toeplitz matvec.

The data plane is libbtg's grid engine (``csrc/btg_grid_engine.cu``, C ABI
``btg_grid_*``): one process per GPU, rank ``i*cols + j`` owns grid cell (i, j)
— the sensors ``[i*ceil(N_d/r), ...)`` x sources ``[j*ceil(N_m/c), ...)``
block of every frequency (the ceiling partition, distributed.cpp:145-175) —
and the per-rank schedule runs in C++ with NCCL on row / column
communicators:

* F  (distributed.cpp:312-351): column broadcast of the parameter slice from
  row 0, local F, row reduce (sum) onto column 0.
* F* (distributed.cpp:353-392): row broadcast of the data slice from column 0,
  local F*, column reduce onto row 0.
* Gauss-Newton Hessian (inverse.cpp:80-85 routed through a partition): the row
  reduce of F and the row broadcast of F* merge into one row all-reduce; Gamma^-1
  is applied in the local C2R epilogue (linear, so before the reduce) and
  alpha R v is added once, on row 0, in the final C2R epilogue.

This module is the Python face of it: :class:`GridEngine` (one rank per
process; ``torch.distributed`` only ships the NCCL unique id), the
single-process :class:`Partition` (the reference's ``Partition`` /
``distributed_forward`` / ``distributed_adjoint`` over a local grid with the P2P
transport), the schedule (:func:`schedule`) and the reference's CommLog byte
model (:func:`comm_events`). ``transport="gloo"`` runs the same C++ schedule
with the collectives handed to torch.distributed/gloo through host callbacks —
it exists so several ranks can share ONE GPU in tests (NCCL refuses duplicate
devices); it is not a compute path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Tuple

from . import _lib
from ._lib import GridError

__all__ = ["Shard", "CommEvent", "partition_bounds", "schedule", "comm_events", "GridEngine",
           "synthetic_shard_operator", "Partition", "partition_operator", "distributed_forward",
           "distributed_adjoint"]


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


@dataclass
class CommEvent:
    """CommEvent (distributed.hpp:77-84)."""

    phase: str
    participants: int
    link_bytes: int
    messages: int
    total_bytes: int
    tree_depth: int


_PHASES = {0: "broadcast", 1: "reduce"}
_KINDS = {"forward": _lib.BTG_GRID_FORWARD, "adjoint": _lib.BTG_GRID_ADJOINT, "hessian": _lib.BTG_GRID_HESSIAN}


def _events(arr, n) -> List[CommEvent]:
    return [CommEvent(_PHASES[e.phase], int(e.participants), int(e.link_bytes), int(e.messages),
                      int(e.total_bytes), int(e.tree_depth)) for e in arr[:n]]


def comm_events(num_sensors: int, num_sources: int, num_steps: int, grid: Tuple[int, int], kind: str):
    """The reference's CommLog of one F ("forward") or F* ("adjoint") over the grid
    (record_collective, distributed.cpp:23-34), from libbtg's model."""
    L = _lib.load()
    cnt = ctypes.c_size_t()
    _lib.check(L.btg_comm_events(num_sensors, num_sources, num_steps, grid[0], grid[1], _KINDS[kind], None, 0,
                                 ctypes.byref(cnt)))
    arr = (_lib.CommEventC * max(1, cnt.value))()
    _lib.check(L.btg_comm_events(num_sensors, num_sources, num_steps, grid[0], grid[1], _KINDS[kind], arr,
                                 cnt.value, ctypes.byref(cnt)))
    return _events(arr, cnt.value)


def schedule(num_sensors: int, num_sources: int, num_steps: int, grid: Tuple[int, int], rank: int, kind: str,
             with_gamma: bool = False, with_reg: bool = False):
    """The per-rank step list the C++ executor runs (btg_grid_schedule), as dicts."""
    L = _lib.load()
    cnt = ctypes.c_size_t()
    args = (num_sensors, num_sources, num_steps, grid[0], grid[1], rank, _KINDS[kind], int(with_gamma),
            int(with_reg))
    _lib.check(L.btg_grid_schedule(*args, None, 0, ctypes.byref(cnt)))
    arr = (_lib.GridStep * max(1, cnt.value))()
    _lib.check(L.btg_grid_schedule(*args, arr, cnt.value, ctypes.byref(cnt)))
    return [{k: int(getattr(st, k)) for k, _ in _lib.GridStep._fields_} for st in arr[:cnt.value]]


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


class _GlooTransport:
    """Host callbacks for btg_grid_create_external over torch.distributed (gloo):
    lets several ranks share one GPU in tests. Every rank creates every row and
    column group in the same order (torch.distributed rule)."""

    def __init__(self, rows: int, cols: int, rank: int):
        import numpy as np
        import torch
        import torch.distributed as dist

        self.rows, self.cols = rows, cols
        self.i, self.j = divmod(rank, cols)
        self._row = [dist.new_group([i * cols + j for j in range(cols)], backend="gloo") for i in range(rows)]
        self._col = [dist.new_group([i * cols + j for i in range(rows)], backend="gloo") for j in range(cols)]

        def view(buf, n):
            return torch.from_numpy(np.ctypeslib.as_array(buf, shape=(n,)))

        def group(g):
            return (self._row[self.i], lambda m: self.i * cols + m) if g == _lib.BTG_GROUP_ROW else \
                   (self._col[self.j], lambda m: m * cols + self.j)

        def bcast(_user, g, buf, n, root):
            try:
                grp, rank_of = group(g)
                dist.broadcast(view(buf, n), src=rank_of(root), group=grp)
                return 0
            except Exception:  # noqa: BLE001 - reported as BTG_ENCCL by the engine
                return 1

        def reduce(_user, g, buf, n, root):
            try:
                grp, rank_of = group(g)
                dist.reduce(view(buf, n), dst=rank_of(root), group=grp)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def allreduce(_user, g, buf, n):
            try:
                grp, _ = group(g)
                dist.all_reduce(view(buf, n), group=grp)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        self.callbacks = _lib.GridCallbacks(None, _lib.BCAST_FN(bcast), _lib.REDUCE_FN(reduce),
                                            _lib.ALLREDUCE_FN(allreduce))


class GridEngine:
    """F / F* / Hessian on an r x c grid of ranks, one GPU each: a thin shim over
    libbtg's ``btg_grid`` (the schedule, the NCCL collectives and the local
    pipelines all run in C++).

    ``local_op`` is this rank's shard (:class:`SpectralOperator`, None for an
    empty shard); the engine borrows it. Vector slices are float64 CUDA tensors
    on the rank's device: parameter slices (local_sources x N_t) on row-0 ranks,
    data slices (local_sensors x N_t) on column-0 ranks, as in the reference
    (scatter_param / scatter_data, distributed.hpp:66-73). Calls run on torch's
    current stream."""

    def __init__(self, num_sensors: int, num_sources: int, num_steps: int, grid: Tuple[int, int], local_op,
                 device=None, transport: str = "nccl"):
        import torch
        import torch.distributed as dist

        self.rows, self.cols = int(grid[0]), int(grid[1])
        self.num_sensors, self.num_sources, self.num_steps = num_sensors, num_sources, num_steps
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        if self.world != self.rows * self.cols:
            raise GridError(f"grid {self.rows}x{self.cols} needs {self.rows * self.cols} ranks, have {self.world}")
        self.shards = partition_bounds(num_sensors, num_sources, self.rows, self.cols)
        self.shard = self.shards[self.rank]
        self.local_op = local_op
        if device is None:
            device = torch.device(f"cuda:{torch.cuda.current_device()}")
        self.device = torch.device(device)
        self.transport = transport
        L = _lib.load()
        h = ctypes.c_void_p()
        dev = self.device.index or 0
        if transport == "nccl":
            uid = ctypes.create_string_buffer(_lib.BTG_NCCL_ID_BYTES)
            if self.rank == 0:
                _lib.check(L.btg_grid_nccl_id(uid))
            obj = [uid.raw if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            _lib.check(L.btg_grid_create(self.rows, self.cols, self.rank, obj[0], dev, ctypes.byref(h)))
        elif transport == "gloo":
            self._gloo = _GlooTransport(self.rows, self.cols, self.rank)
            _lib.check(L.btg_grid_create_external(self.rows, self.cols, self.rank, dev,
                                                  ctypes.byref(self._gloo.callbacks), ctypes.byref(h)))
        else:
            raise _lib.Error(f"unknown grid transport '{transport}' (nccl or gloo)")
        self._h = h
        try:
            _lib.check(L.btg_grid_set_dims(h, num_sensors, num_sources, num_steps))
            _lib.check(L.btg_grid_attach(h, self.rank, local_op._h if local_op is not None else None, 0))
        except Exception:
            L.btg_grid_destroy(h)
            self._h = None
            raise

    # -- construction helpers ---------------------------------------------------
    @classmethod
    def synthetic(cls, num_sensors: int, num_sources: int, num_steps: int, grid: Tuple[int, int], seed: int,
                  precision: int = 64, transport: str = "nccl"):
        """Each rank builds its own shard of the synthetic operator on its GPU."""
        import torch
        import torch.distributed as dist

        rank = dist.get_rank()
        shard = partition_bounds(num_sensors, num_sources, *grid)[rank]
        device = torch.cuda.current_device()
        op = None if shard.empty else synthetic_shard_operator(num_sensors, num_sources, num_steps, shard, seed,
                                                               device, precision)
        return cls(num_sensors, num_sources, num_steps, grid, op, device=torch.device(f"cuda:{device}"),
                   transport=transport)

    @classmethod
    def from_blocks(cls, blocks, grid: Tuple[int, int], precision: int = 64, transport: str = "nccl"):
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
        return cls(nd, nm, nt, grid, op, device=torch.device(f"cuda:{device}"), transport=transport)

    @classmethod
    def from_file(cls, path, grid: Tuple[int, int], precision: int = 64, transport: str = "nccl"):
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
        return cls(nd, nm, nt, grid, op, device=torch.device(f"cuda:{device}"), transport=transport)

    @classmethod
    def from_operator(cls, op, grid: Tuple[int, int], transport: str = "nccl"):
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
        return cls(nd, nm, nt, grid, local, device=torch.device(f"cuda:{device}"), transport=transport)

    @staticmethod
    def plan(num_sensors: int, num_sources: int, workers: Optional[int] = None,
             gpus_per_node: int = 1) -> Tuple[int, int]:
        """The planner's grid for the world size (or ``workers``)."""
        from .planner import plan_grid

        if workers is None:
            import torch.distributed as dist

            workers = dist.get_world_size()
        return plan_grid(num_sensors, num_sources, workers, gpus_per_node)

    # -- helpers -------------------------------------------------------------------
    def param_slice_bounds(self, j: int) -> Tuple[int, int]:
        s = self.shards[j]
        return s.source_begin, s.source_end

    def data_slice_bounds(self, i: int) -> Tuple[int, int]:
        s = self.shards[i * self.cols]
        return s.sensor_begin, s.sensor_end

    def _slice_in(self, x, dim: int, owner: bool, what: str):
        import torch

        if not owner:
            return None
        if x is None:
            raise ValueError(f"{what}: this rank owns a slice and must pass it")
        if tuple(x.shape) != (dim, self.num_steps):
            raise _lib.DimensionError(f"{what}: slice is {tuple(x.shape)}, expected ({dim}, {self.num_steps})")
        if not isinstance(x, torch.Tensor) or x.device != self.device or x.dtype != torch.float64:
            raise _lib.Error(f"{what}: slices are float64 tensors on {self.device}")
        return x.contiguous()

    def _bind(self):
        import torch

        s = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(_lib.load().btg_grid_set_stream(self._h, s or _lib.CUDA_STREAM_LEGACY))

    def _call(self, kind: str, x, din: int, dout: int, in_owner: bool, out_owner: bool, extra=()):
        import torch

        xin = self._slice_in(x, din, in_owner, kind)
        out = torch.empty((dout, self.num_steps), dtype=torch.float64, device=self.device) if out_owner else None
        self._bind()
        L = _lib.load()
        fn = {"forward": L.btg_grid_forward, "adjoint": L.btg_grid_adjoint, "hessian": L.btg_grid_hessian}[kind]
        args = [self._h, xin.data_ptr() if xin is not None else None, xin.numel() if xin is not None else 0,
                out.data_ptr() if out is not None else None, out.numel() if out is not None else 0]
        _lib.check(fn(*args, *extra, _lib.BTG_DEVICE_PTRS))
        return out

    # -- the three actions ---------------------------------------------------------
    def forward(self, m_slice=None):
        """distributed_forward (distributed.cpp:312-351). Row-0 ranks pass their
        parameter slice; column-0 ranks get their data slice back (else None)."""
        sh = self.shard
        return self._call("forward", m_slice, sh.local_sources, sh.local_sensors, sh.grid_row == 0,
                          sh.grid_col == 0)

    def adjoint(self, d_slice=None):
        """distributed_adjoint (distributed.cpp:353-392). Column-0 ranks pass
        their data slice; row-0 ranks get their parameter slice back."""
        sh = self.shard
        return self._call("adjoint", d_slice, sh.local_sensors, sh.local_sources, sh.grid_col == 0,
                          sh.grid_row == 0)

    def hessian(self, v_slice=None, alpha: float = 0.0, reg="identity", gamma_inv=None):
        """F* Gamma^-1 F v + alpha R v over the grid; row-0 ranks pass and receive
        parameter slices. gamma_inv is GLOBAL ((N_d,) or (N_d, N_t), on the
        rank's device) and the same on every rank."""
        import torch

        from .operator import _REG

        rk = _REG.get(reg)
        if rk is None:
            raise _lib.Error(f"unknown regularization '{reg}'")
        gk, gp = _lib.BTG_GAMMA_NONE, None
        if gamma_inv is not None:
            if not isinstance(gamma_inv, torch.Tensor) or gamma_inv.device != self.device:
                raise _lib.Error(f"hessian: gamma_inv must be a tensor on {self.device}")
            g = gamma_inv.contiguous()
            if tuple(g.shape) == (self.num_sensors,):
                gk = _lib.BTG_GAMMA_PER_SENSOR
            elif tuple(g.shape) == (self.num_sensors, self.num_steps):
                gk = _lib.BTG_GAMMA_PER_SAMPLE
            else:
                raise _lib.DimensionError(f"hessian: gamma_inv must be ({self.num_sensors},) or "
                                          f"({self.num_sensors}, {self.num_steps}) (global)")
            gp = g.data_ptr()
            self._gkeep = g
        sh = self.shard
        return self._call("hessian", v_slice, sh.local_sources, sh.local_sources, sh.grid_row == 0,
                          sh.grid_row == 0, extra=(gp, gk, float(alpha), rk))

    def synchronize(self):
        _lib.check(_lib.load().btg_grid_synchronize(self._h))

    @property
    def comm_log(self) -> List[CommEvent]:
        L = _lib.load()
        cnt = ctypes.c_size_t()
        _lib.check(L.btg_grid_comm_log(self._h, None, 0, ctypes.byref(cnt)))
        arr = (_lib.CommEventC * max(1, cnt.value))()
        _lib.check(L.btg_grid_comm_log(self._h, arr, cnt.value, ctypes.byref(cnt)))
        return _events(arr, cnt.value)

    def comm_bytes(self) -> int:
        return sum(e.total_bytes for e in self.comm_log)

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().btg_grid_destroy(self._h)
            self._h = None
        if self.local_op is not None and hasattr(self.local_op, "close"):
            self.local_op.close()
        self.local_op = None

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.load().btg_grid_destroy(self._h)
                self._h = None
        except Exception:
            pass


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

    def hessian(self, v, alpha: float = 0.0, reg="identity", gamma_inv=None, backend: str = "fft",
                parallel: bool = False):
        """HessianOperator::apply with this partition (inverse.cpp:78-91), plus a
        global Gamma^-1 ((N_d,) or (N_d, N_t)): the grid Hessian schedule."""
        import numpy as np

        from .operator import _REG

        rk = _REG.get(reg)
        if rk is None:
            raise _lib.Error(f"unknown regularization '{reg}'")
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.shape != (self.num_sources, self.num_steps):
            raise _lib.DimensionError(f"hessian: vector is {v.shape}, expected ({self.num_sources}, {self.num_steps})")
        gk, gp, g = _lib.BTG_GAMMA_NONE, None, None
        if gamma_inv is not None:
            g = np.ascontiguousarray(gamma_inv, dtype=np.float64)
            if g.shape == (self.num_sensors,):
                gk = _lib.BTG_GAMMA_PER_SENSOR
            elif g.shape == (self.num_sensors, self.num_steps):
                gk = _lib.BTG_GAMMA_PER_SAMPLE
            else:
                raise _lib.DimensionError("hessian: gamma_inv has the wrong shape")
            gp = g.ctypes.data
        out = np.empty_like(v)
        _lib.check(_lib.load().btg_partition_hessian(self._h, v.ctypes.data, v.size, out.ctypes.data, out.size, gp,
                                                     gk, float(alpha), rk, _parse_backend(backend),
                                                     int(bool(parallel))))
        return out

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
