"""ctypes binding of ``libbtg.so`` (the C ABI declared in ``include/btg.h``).

There is deliberately no fallback: if the CUDA library is missing or no GPU is
visible, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libbtg.so"

BTG_OK, BTG_EDIM, BTG_EORDER, BTG_EARG, BTG_ECUDA, BTG_ENOMEM, BTG_EGRID, BTG_ESOLVER, BTG_EFORMAT = range(9)
BTG_F64, BTG_F32 = 64, 32
BTG_DEVICE_PTRS = 0x1
BTG_KEEP_CHANNEL_LAYOUT = 0x2
CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: the legacy default stream (torch's stream 0)
BTG_REG_IDENTITY, BTG_REG_TEMPORAL_LAPLACIAN = 0, 1
BTG_GAMMA_NONE, BTG_GAMMA_PER_SENSOR, BTG_GAMMA_PER_SAMPLE = 0, 1, 2

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
    "btg_partition_destroy",
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
    for name in EXPORTED:
        if name not in ("btg_last_error", "btg_abi_version", "btg_destroy", "btg_apply_arithmetic_intensity",
                        "btg_partition_destroy"):
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
    raise Error(msg)
