"""ctypes binding of ``libbtg.so`` (the C ABI declared in ``include/btg.h``).

There is deliberately no fallback: if the CUDA library is missing or no GPU is
visible, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libbtg.so"

BTG_OK, BTG_EDIM, BTG_EORDER, BTG_EARG, BTG_ECUDA, BTG_ENOMEM, BTG_EGRID, BTG_ESOLVER, BTG_EFORMAT, BTG_ENCCL = range(10)
BTG_F64, BTG_F32 = 64, 32
BTG_DEVICE_PTRS = 0x1
BTG_KEEP_CHANNEL_LAYOUT = 0x2
CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: the legacy default stream (torch's stream 0)
BTG_REG_IDENTITY, BTG_REG_TEMPORAL_LAPLACIAN = 0, 1
BTG_GAMMA_NONE, BTG_GAMMA_PER_SENSOR, BTG_GAMMA_PER_SAMPLE = 0, 1, 2
BTG_GRID_FORWARD, BTG_GRID_ADJOINT, BTG_GRID_HESSIAN = 0, 1, 2
(BTG_STEP_INPUT, BTG_STEP_BROADCAST, BTG_STEP_FORWARD, BTG_STEP_ADJOINT, BTG_STEP_REDUCE, BTG_STEP_ALLREDUCE,
 BTG_STEP_OUTPUT) = range(7)
BTG_GROUP_ROW, BTG_GROUP_COL = 0, 1
BTG_TRANSPORT_NCCL, BTG_TRANSPORT_P2P, BTG_TRANSPORT_EXTERNAL = 0, 1, 2
BTG_NCCL_ID_BYTES = 128

# Every symbol include/btg.h declares (checked by tests/test_abi.py).
EXPORTED = (
    "btg_last_error",
    "btg_abi_version",
    "btg_create",
    "btg_setup_rows",
    "btg_setup",
    "btg_forward",
    "btg_adjoint",
    "btg_hessian",
    "btg_set_stream",
    "btg_synchronize",
    "btg_set_timing",
    "btg_set_multi_rhs_engine",
    "btg_set_channel_layout",
    "btg_has_channel_layout",
    "btg_forward_ewp",
    "btg_naive_forward",
    "btg_write_compact",
    "btg_partition_create",
    "btg_partition_from_operator",
    "btg_partition_shard",
    "btg_partition_forward",
    "btg_partition_adjoint",
    "btg_partition_hessian",
    "btg_partition_destroy",
    "btg_grid_schedule",
    "btg_comm_events",
    "btg_grid_nccl_id",
    "btg_grid_create",
    "btg_grid_create_local",
    "btg_grid_create_external",
    "btg_grid_set_dims",
    "btg_grid_setup",
    "btg_grid_from_operator",
    "btg_grid_attach",
    "btg_grid_shard",
    "btg_grid_info",
    "btg_grid_forward",
    "btg_grid_adjoint",
    "btg_grid_hessian",
    "btg_grid_set_backend",
    "btg_grid_set_stream",
    "btg_grid_synchronize",
    "btg_grid_comm_log",
    "btg_grid_reset_comm_log",
    "btg_grid_destroy",
    "btg_read_compact",
    "btg_conventional_cost_estimate",
    "btg_apply_arithmetic_intensity",
    "btg_naive_adjoint",
    "btg_adjoint_ewp",
    "btg_get_counters",
    "btg_reset_counters",
    "btg_get_dims",
    "btg_export_spectrum",
    "btg_spectrum_device",
    "btg_destroy",
    "btg_fill_uniform",
    "btg_forward_ex",
    "btg_adjoint_ex",
    "btg_fill_uniform_3d",
    "btg_cg_solve",
    "btg_objective",
    "btg_export_spectrum_block",
    "btg_peek_operator",
    "btg_load_operator",
    "btg_save_operator",
    "btg_write_vector",
    "btg_read_vector",
    "btg_load_operator_rect",
    "btg_slice_operator",
    "btg_select_grid",
    "btg_weak_scaling_shape",
    "btg_modified_cost",
    "btg_comm_cost",
    "btg_default_hw_model",
    "btg_plan_grid",
)


class Error(RuntimeError):
    """btoep::Error (errors.hpp:8-10) / CUDA failure."""


class DimensionError(ValueError):
    """btoep::DimensionError (errors.hpp:13-15)."""


class OrderingError(ValueError):
    """btoep::OrderingError (errors.hpp:18-20)."""


class GridError(ValueError):
    """btoep::GridError (errors.hpp:28-30)."""


class SolverError(RuntimeError):
    """btoep::SolverError (errors.hpp:33-35); the reference binds it to RuntimeError."""


class FormatError(ValueError):
    """btoep::FormatError (errors.hpp:23-25)."""


class CommError(RuntimeError):
    """NCCL / grid transport failure (BTG_ENCCL)."""


class FileHeader(ctypes.Structure):
    """btg_file_header == io::OperatorHeader (io.hpp:21-28)."""

    _fields_ = [
        ("ordering", ctypes.c_int),
        ("domain", ctypes.c_int),
        ("num_sensors", ctypes.c_uint64),
        ("num_sources", ctypes.c_uint64),
        ("num_steps", ctypes.c_uint64),
        ("complex_scalar", ctypes.c_int),
    ]


class CgResult(ctypes.Structure):
    """btg_cg_result == btoep::CGResult minus the solution (inverse.hpp:44-49)."""

    _fields_ = [
        ("iterations", ctypes.c_size_t),
        ("relative_residual", ctypes.c_double),
        ("converged", ctypes.c_int),
        ("seconds", ctypes.c_double),
    ]


class Epilogue(ctypes.Structure):
    """btg_epilogue: fused Gamma^-1 / alpha R v store epilogue."""

    _fields_ = [
        ("gamma_inv", ctypes.c_void_p),
        ("gamma_kind", ctypes.c_int),
        ("reg_v", ctypes.c_void_p),
        ("alpha", ctypes.c_double),
        ("reg_kind", ctypes.c_int),
    ]


class GridStep(ctypes.Structure):
    """btg_grid_step: one step of a rank's grid schedule."""

    _fields_ = [
        ("op", ctypes.c_int),
        ("group", ctypes.c_int),
        ("root", ctypes.c_int),
        ("src", ctypes.c_int),
        ("dst", ctypes.c_int),
        ("active", ctypes.c_int),
        ("gamma", ctypes.c_int),
        ("reg", ctypes.c_int),
        ("count", ctypes.c_size_t),
    ]


class CommEventC(ctypes.Structure):
    """btg_comm_event == btoep::CommEvent (distributed.hpp:77-84)."""

    _fields_ = [
        ("phase", ctypes.c_int),
        ("participants", ctypes.c_size_t),
        ("messages", ctypes.c_size_t),
        ("link_bytes", ctypes.c_uint64),
        ("total_bytes", ctypes.c_uint64),
        ("tree_depth", ctypes.c_size_t),
    ]


BCAST_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                            ctypes.c_size_t, ctypes.c_int)
REDUCE_FN = BCAST_FN
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                ctypes.c_size_t)


class GridCallbacks(ctypes.Structure):
    """btg_grid_callbacks: host-callback transport (tests)."""

    _fields_ = [
        ("user", ctypes.c_void_p),
        ("broadcast", BCAST_FN),
        ("reduce", REDUCE_FN),
        ("allreduce", ALLREDUCE_FN),
    ]


class HwModel(ctypes.Structure):
    """btg_hw_model: rates of the B200 / NVSwitch planner."""

    _fields_ = [
        ("hbm_gbs", ctypes.c_double),
        ("fft_gbs", ctypes.c_double),
        ("link_gbs", ctypes.c_double),
        ("node_link_gbs", ctypes.c_double),
        ("latency_us", ctypes.c_double),
        ("gpus_per_node", ctypes.c_uint),
    ]


class GridPlan(ctypes.Structure):
    """btg_grid_plan: modelled seconds of one action on an r x c grid."""

    _fields_ = [
        ("rows", ctypes.c_size_t),
        ("cols", ctypes.c_size_t),
        ("seconds", ctypes.c_double),
        ("local_seconds", ctypes.c_double),
        ("comm_seconds", ctypes.c_double),
    ]


class _Stage(ctypes.Structure):
    _fields_ = [("ops", ctypes.c_double), ("bytes", ctypes.c_double), ("seconds", ctypes.c_double)]


class Counters(ctypes.Structure):
    """btg_counters == btoep::PipelineCounters stages (counters.hpp:18-45)."""

    _fields_ = [
        ("pad", _Stage),
        ("forward_fft", _Stage),
        ("reorder_in", _Stage),
        ("apply", _Stage),
        ("reorder_out", _Stage),
        ("inverse_fft", _Stage),
        ("unpad", _Stage),
        ("launches", ctypes.c_uint64),
    ]

    def as_dict(self):
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            out[name] = v if isinstance(v, int) else {"ops": v.ops, "bytes": v.bytes, "seconds": v.seconds}
        return out


_lib = None
_sz = ctypes.c_size_t
_vp = ctypes.c_void_p
_dp = ctypes.c_void_p  # pointers passed as integers (host or device)


def load():
    """Load libbtg.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise Error(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    L.btg_last_error.restype = ctypes.c_char_p
    L.btg_abi_version.restype = ctypes.c_int
    L.btg_create.argtypes = [_sz, _sz, _sz, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]
    L.btg_setup_rows.argtypes = [_vp, _dp, _sz, _sz, ctypes.c_uint]
    L.btg_setup.argtypes = [_dp, _sz, _sz, _sz, ctypes.c_int, ctypes.c_int, ctypes.c_uint, ctypes.POINTER(_vp)]
    L.btg_forward.argtypes = [_vp, _dp, _sz, _dp, _sz, _sz, ctypes.c_uint]
    L.btg_adjoint.argtypes = [_vp, _dp, _sz, _dp, _sz, _sz, ctypes.c_uint]
    L.btg_hessian.argtypes = [_vp, _dp, _sz, _dp, _sz, _sz, _dp, ctypes.c_int, ctypes.c_double,
                              ctypes.c_int, ctypes.c_uint]
    L.btg_set_stream.argtypes = [_vp, _vp]
    L.btg_synchronize.argtypes = [_vp]
    L.btg_set_timing.argtypes = [_vp, ctypes.c_int]
    L.btg_set_multi_rhs_engine.argtypes = [_vp, ctypes.c_int]
    L.btg_set_channel_layout.argtypes = [_vp, ctypes.c_int]
    L.btg_has_channel_layout.argtypes = [_vp, ctypes.POINTER(ctypes.c_int)]
    L.btg_forward_ewp.argtypes = [_vp, _dp, _sz, _dp, _sz, ctypes.c_uint]
    L.btg_conventional_cost_estimate.argtypes = [ctypes.c_double] * 4 + [ctypes.POINTER(ctypes.c_double * 7)]
    L.btg_apply_arithmetic_intensity.argtypes = [ctypes.c_double, ctypes.c_double]
    L.btg_apply_arithmetic_intensity.restype = ctypes.c_double
    L.btg_partition_create.argtypes = [_dp, _sz, _sz, _sz, _sz, _sz, ctypes.POINTER(ctypes.c_int), _sz,
                                       ctypes.c_int, ctypes.c_uint, ctypes.POINTER(_vp)]
    L.btg_partition_from_operator.argtypes = [_vp, _sz, _sz, ctypes.POINTER(ctypes.c_int), _sz, ctypes.POINTER(_vp)]
    L.btg_partition_shard.argtypes = [_vp, _sz, _sz, ctypes.POINTER(_sz), ctypes.POINTER(_vp)]
    for name in ("btg_partition_forward", "btg_partition_adjoint"):
        getattr(L, name).argtypes = [_vp, _dp, _sz, _dp, _sz, ctypes.c_int, ctypes.c_int]
    L.btg_partition_hessian.argtypes = [_vp, _dp, _sz, _dp, _sz, _dp, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int]
    L.btg_grid_schedule.argtypes = [_sz, _sz, _sz, _sz, _sz, _sz, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(GridStep), _sz, ctypes.POINTER(_sz)]
    L.btg_comm_events.argtypes = [_sz, _sz, _sz, _sz, _sz, ctypes.c_int, ctypes.POINTER(CommEventC), _sz,
                                  ctypes.POINTER(_sz)]
    L.btg_grid_nccl_id.argtypes = [ctypes.c_char_p]
    L.btg_grid_create.argtypes = [_sz, _sz, _sz, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(_vp)]
    L.btg_grid_create_local.argtypes = [_sz, _sz, ctypes.POINTER(ctypes.c_int), _sz, ctypes.c_int,
                                        ctypes.POINTER(_vp)]
    L.btg_grid_create_external.argtypes = [_sz, _sz, _sz, ctypes.c_int, ctypes.POINTER(GridCallbacks),
                                           ctypes.POINTER(_vp)]
    L.btg_grid_set_dims.argtypes = [_vp, _sz, _sz, _sz]
    L.btg_grid_setup.argtypes = [_vp, _dp, _sz, _sz, _sz, ctypes.c_int, ctypes.c_uint]
    L.btg_grid_from_operator.argtypes = [_vp, _vp]
    L.btg_grid_attach.argtypes = [_vp, _sz, _vp, ctypes.c_int]
    L.btg_grid_shard.argtypes = [_vp, _sz, ctypes.POINTER(_sz), ctypes.POINTER(_vp)]
    L.btg_grid_info.argtypes = [_vp, ctypes.POINTER(_sz), ctypes.POINTER(_sz), ctypes.POINTER(_sz),
                                ctypes.POINTER(ctypes.c_int)]
    for name in ("btg_grid_forward", "btg_grid_adjoint"):
        getattr(L, name).argtypes = [_vp, _dp, _sz, _dp, _sz, ctypes.c_uint]
    L.btg_grid_hessian.argtypes = [_vp, _dp, _sz, _dp, _sz, _dp, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                   ctypes.c_uint]
    L.btg_grid_set_backend.argtypes = [_vp, ctypes.c_int, ctypes.c_int]
    L.btg_grid_set_stream.argtypes = [_vp, _vp]
    L.btg_grid_synchronize.argtypes = [_vp]
    L.btg_grid_comm_log.argtypes = [_vp, ctypes.POINTER(CommEventC), _sz, ctypes.POINTER(_sz)]
    L.btg_grid_reset_comm_log.argtypes = [_vp]
    L.btg_grid_destroy.argtypes = [_vp]
    L.btg_grid_destroy.restype = None
    L.btg_partition_destroy.argtypes = [_vp]
    L.btg_partition_destroy.restype = None
    L.btg_write_compact.argtypes = [ctypes.c_char_p, _dp, _sz, _sz, _sz]
    L.btg_read_compact.argtypes = [ctypes.c_char_p, _dp, _sz, ctypes.POINTER(_sz), ctypes.POINTER(_sz),
                                   ctypes.POINTER(_sz)]
    for name in ("btg_naive_forward", "btg_naive_adjoint"):
        getattr(L, name).argtypes = [_dp, _sz, _sz, _sz, _dp, _dp, ctypes.c_int, ctypes.c_uint]
    L.btg_adjoint_ewp.argtypes = [_vp, _dp, _sz, _dp, _sz, ctypes.c_uint]
    L.btg_get_counters.argtypes = [_vp, ctypes.POINTER(Counters)]
    L.btg_reset_counters.argtypes = [_vp]
    L.btg_get_dims.argtypes = [_vp, ctypes.POINTER(_sz), ctypes.POINTER(_sz), ctypes.POINTER(_sz),
                               ctypes.POINTER(ctypes.c_int)]
    L.btg_export_spectrum.argtypes = [_vp, _dp, ctypes.c_int]
    L.btg_spectrum_device.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_sz)]
    L.btg_destroy.argtypes = [_vp]
    L.btg_destroy.restype = None
    L.btg_fill_uniform.argtypes = [_dp, _sz, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double,
                                   ctypes.c_double, _vp]
    L.btg_forward_ex.argtypes = [_vp, _dp, _sz, _dp, _sz, _sz, ctypes.POINTER(Epilogue), ctypes.c_uint]
    L.btg_adjoint_ex.argtypes = [_vp, _dp, _sz, _dp, _sz, _sz, ctypes.POINTER(Epilogue), ctypes.c_uint]
    L.btg_fill_uniform_3d.argtypes = [_dp, _sz, _sz, _sz, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_double, ctypes.c_double, _vp]
    L.btg_cg_solve.argtypes = [_vp, _dp, _sz, _dp, _sz, _dp, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                               ctypes.c_double, _sz, ctypes.c_int, ctypes.c_uint, ctypes.POINTER(CgResult)]
    L.btg_objective.argtypes = [_vp, _dp, _sz, _dp, _sz, ctypes.c_double, ctypes.c_int, ctypes.c_uint,
                                ctypes.POINTER(ctypes.c_double)]
    L.btg_export_spectrum_block.argtypes = [_vp, _sz, _dp]
    L.btg_peek_operator.argtypes = [ctypes.c_char_p, ctypes.POINTER(FileHeader)]
    L.btg_load_operator.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]
    L.btg_save_operator.argtypes = [_vp, ctypes.c_char_p]
    L.btg_load_operator_rect.argtypes = [ctypes.c_char_p, _sz, _sz, _sz, _sz, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(_vp)]
    L.btg_write_vector.argtypes = [ctypes.c_char_p, _dp, _sz, _sz, ctypes.c_int]
    L.btg_read_vector.argtypes = [ctypes.c_char_p, _dp, _sz, ctypes.POINTER(_sz), ctypes.POINTER(_sz),
                                  ctypes.POINTER(ctypes.c_int)]
    L.btg_slice_operator.argtypes = [_vp, _sz, _sz, _sz, _sz, ctypes.c_int, ctypes.POINTER(_vp)]
    L.btg_select_grid.argtypes = [_sz, ctypes.c_double, ctypes.c_uint, ctypes.POINTER(_sz), ctypes.POINTER(_sz)]
    L.btg_weak_scaling_shape.argtypes = [ctypes.c_double, _sz, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_sz),
                                         ctypes.POINTER(_sz)]
    L.btg_modified_cost.argtypes = [ctypes.c_double, _sz, ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
    L.btg_comm_cost.argtypes = [_sz, _sz, _sz, _sz, _sz, ctypes.c_double, ctypes.c_double,
                                ctypes.POINTER(ctypes.c_double)]
    L.btg_default_hw_model.argtypes = [ctypes.POINTER(HwModel)]
    L.btg_plan_grid.argtypes = [_sz, _sz, _sz, _sz, ctypes.c_int, ctypes.c_int, ctypes.POINTER(HwModel),
                                ctypes.POINTER(GridPlan), ctypes.POINTER(GridPlan), _sz, ctypes.POINTER(_sz)]
    for name in EXPORTED:
        if name not in ("btg_last_error", "btg_abi_version", "btg_destroy", "btg_apply_arithmetic_intensity",
                        "btg_partition_destroy", "btg_grid_destroy"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def check(status: int) -> None:
    """Map a btg_status to the reference's exception taxonomy (errors.hpp)."""
    if status == BTG_OK:
        return
    msg = load().btg_last_error().decode(errors="replace")
    if status == BTG_EDIM:
        raise DimensionError(msg)
    if status == BTG_EORDER:
        raise OrderingError(msg)
    if status == BTG_EGRID:
        raise GridError(msg)
    if status == BTG_ENOMEM:
        raise MemoryError(msg)
    if status == BTG_ESOLVER:
        raise SolverError(msg)
    if status == BTG_EFORMAT:
        raise FormatError(msg)
    if status == BTG_ENCCL:
        raise CommError(msg)
    raise Error(msg)
