"""The reference's operator / vector files.

Mirrors ``btoep::io`` (``proj/include/btoep/io.hpp``, ``src/io.cpp``) and the
reference binding's ``read_vector`` / ``write_vector`` (numpy ``(spatial,
steps)`` SOTI arrays). Operator files go straight between disk and HBM:
``load_operator`` builds the device operator from a time-domain file (setup,
streamed in sensor-row slabs) or a frequency-domain file (the N_t+1 stored
blocks); ``save_operator`` writes the reference's 2 N_t frequency-domain file.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

from . import _lib
from ._lib import check
from .operator import SpectralOperator

__all__ = ["peek_operator", "load_operator", "load_operator_rect", "save_operator", "read_vector", "write_vector",
           "read_operator", "write_operator"]


def peek_operator(path) -> dict:
    """io::peek_operator (io.cpp:132-157)."""
    h = _lib.FileHeader()
    check(_lib.load().btg_peek_operator(str(Path(path)).encode(), ctypes.byref(h)))
    return {"ordering": "TOSI" if h.ordering == 0 else "SOTI", "domain": "time" if h.domain == 0 else "frequency",
            "num_sensors": h.num_sensors, "num_sources": h.num_sources, "num_steps": h.num_steps,
            "complex_scalar": bool(h.complex_scalar)}


def load_operator(path, precision: int = 64, device: int = 0) -> SpectralOperator:
    """The CLI's load_operator (tools/main.cpp:187-203) onto the GPU."""
    h = ctypes.c_void_p()
    check(_lib.load().btg_load_operator(str(Path(path)).encode(), int(precision), int(device), ctypes.byref(h)))
    nd, nm, nt = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    prec = ctypes.c_int()
    check(_lib.load().btg_get_dims(h, ctypes.byref(nd), ctypes.byref(nm), ctypes.byref(nt), ctypes.byref(prec)))
    return SpectralOperator(h.value, nd.value, nm.value, nt.value, prec.value, int(device))


def load_operator_rect(path, sensors, sources, precision: int = 64, device: int = 0) -> SpectralOperator:
    """One grid cell's shard, sensors [i0, i1) x sources [j0, j1), of an operator
    file (btg_load_operator_rect): setup of the rectangle for a time-domain file,
    the rectangle of the stored blocks (no re-setup) for a frequency-domain one."""
    (i0, i1), (j0, j1) = sensors, sources
    h = ctypes.c_void_p()
    check(_lib.load().btg_load_operator_rect(str(Path(path)).encode(), i0, i1, j0, j1, int(precision), int(device),
                                             ctypes.byref(h)))
    return SpectralOperator(h.value, i1 - i0, j1 - j0, peek_operator(path)["num_steps"], int(precision), int(device))


def save_operator(op: SpectralOperator, path) -> None:
    """io::write_operator(SpectralP2O) (io.cpp:113-130), 2 N_t frequencies."""
    check(_lib.load().btg_save_operator(op._h, str(Path(path)).encode()))


def write_vector(path, values, ordering: str = "SOTI") -> None:
    """io::write_vector (io.cpp:207-217); values is (spatial, steps) for SOTI,
    (steps, spatial) for TOSI — the binding's convention (bindings.cpp:48-60)."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.ndim != 2:
        raise _lib.DimensionError("vector must be 2-D")
    if ordering == "SOTI":
        sp, st, o = v.shape[0], v.shape[1], 1
    elif ordering == "TOSI":
        st, sp, o = v.shape[0], v.shape[1], 0
    else:
        raise _lib.OrderingError(f"unknown ordering {ordering!r}")
    check(_lib.load().btg_write_vector(str(Path(path)).encode(), v.ctypes.data, sp, st, o))


def read_vector(path) -> np.ndarray:
    """io::read_vector (io.cpp:219-240), returned as a (spatial, steps) SOTI array."""
    L = _lib.load()
    sp, st = ctypes.c_size_t(), ctypes.c_size_t()
    o = ctypes.c_int()
    p = str(Path(path)).encode()
    check(L.btg_read_vector(p, None, 0, ctypes.byref(sp), ctypes.byref(st), ctypes.byref(o)))
    flat = np.empty(sp.value * st.value, dtype=np.float64)
    check(L.btg_read_vector(p, flat.ctypes.data, flat.size, None, None, None))
    if o.value == 1:
        return flat.reshape(sp.value, st.value)
    return np.ascontiguousarray(flat.reshape(st.value, sp.value).T)


def write_operator(path, blocks) -> None:
    """The reference module's write_operator(path, blocks) (bindings.cpp:306-310,
    io.cpp:97-111): a time-domain TOSI file of (steps, sensors, sources) blocks."""
    b = np.ascontiguousarray(blocks, dtype=np.float64)
    if b.ndim != 3:
        raise _lib.DimensionError("blocks must be (steps, sensors, sources)")
    nt, nd, nm = b.shape
    check(_lib.load().btg_write_compact(str(Path(path)).encode(), b.ctypes.data, nd, nm, nt))


def read_operator(path) -> np.ndarray:
    """read_operator(path) (bindings.cpp:311-315, io.cpp:159-180): the compact
    (steps, sensors, sources) blocks of a time-domain file; FormatError for a
    frequency-domain one."""
    L = _lib.load()
    p = str(Path(path)).encode()
    nd, nm, nt = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    check(L.btg_read_compact(p, None, 0, ctypes.byref(nd), ctypes.byref(nm), ctypes.byref(nt)))
    out = np.empty((nt.value, nd.value, nm.value), dtype=np.float64)
    check(L.btg_read_compact(p, out.ctypes.data, out.size, None, None, None))
    return out

