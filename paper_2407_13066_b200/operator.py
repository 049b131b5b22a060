"""Host-side mirror of the reference's operator API over the C ABI.

Same names, argument meaning and error behaviour as the reference's Python
module (``/root/reference/proj/python/src/bindings.cpp``):

* ``setup(blocks)`` — blocks are ``(steps, sensors, sources)`` float64
  (bindings.cpp:34-39, 126-132); returns a :class:`SpectralOperator`.
* ``SpectralOperator.apply_forward(m)`` / ``apply_adjoint(d)`` — vectors are
  ``(spatial, steps)`` SOTI arrays (bindings.cpp:101-112); a leading batch
  axis ``(nrhs, spatial, steps)`` selects the multi-right-hand-side path.
* ``HessianOperator(op, alpha, reg).apply(v)`` — inverse.hpp:32-39, plus the
  north star's noise weighting ``gamma_inv``.
* Shape errors raise :class:`DimensionError` (a ``ValueError``, as the
  reference's bindings register it, bindings.cpp:81-85).

numpy inputs go through host buffers (the reference's by-value semantics);
CUDA ``torch.Tensor`` inputs stay on the device and return device tensors,
ordered on torch's current stream.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _lib
from ._lib import BTG_DEVICE_PTRS, BTG_F32, BTG_F64, DimensionError, check

__all__ = ["SpectralOperator", "HessianOperator", "setup", "create", "fill_uniform"]

_REG = {"identity": 0, "scaled-identity": 0, "temporal-laplacian": 1, 0: 0, 1: 1}


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch") and hasattr(x, "data_ptr")


def _torch_stream_ptr(t) -> int:
    import torch

    return torch.cuda.current_stream(t.device).cuda_stream


class SpectralOperator:
    """Device-resident frequency-domain operator (the reference's SpectralP2O,
    block_operator.hpp:36-55). F-hat holds the N_t+1 non-redundant frequencies;
    ``num_freq`` reports the reference's 2*N_t for API parity."""

    def __init__(self, handle: int, nd: int, nm: int, nt: int, precision: int, device: int):
        self._h = ctypes.c_void_p(handle)
        self.num_sensors, self.num_sources, self.num_steps = nd, nm, nt
        self.precision = precision
        self.device = device

    # -- reference surface ----------------------------------------------------
    @property
    def num_freq(self) -> int:
        return 2 * self.num_steps

    @property
    def num_stored_freq(self) -> int:
        return self.num_steps + 1

    @property
    def freq_blocks(self) -> np.ndarray:
        """The reference's (2*steps, sensors, sources) complex spectrum
        (bindings.cpp:91-99), rebuilt from the stored half by conjugate symmetry."""
        return self.spectrum(full=True)

    def spectrum(self, full: bool = False) -> np.ndarray:
        nf = 2 * self.num_steps if full else self.num_steps + 1
        out = np.empty((nf, self.num_sensors, self.num_sources), dtype=np.complex128)
        check(_lib.load().btg_export_spectrum(self._h, out.ctypes.data, int(full)))
        return out

    def apply_forward(self, m, gamma_inv=None):
        """d = F m (block_operator.cpp:218-273); with ``gamma_inv`` the output is
        weighted by Gamma^-1 in the fused C2R epilogue (d = Gamma^-1 F m)."""
        return self._apply(m, adjoint=False, gamma_inv=gamma_inv)

    def apply_adjoint(self, d, reg_v=None, alpha: float = 0.0, reg="identity"):
        """m = F* d (block_operator.cpp:275-331); with ``reg_v`` and ``alpha`` the
        fused epilogue adds alpha R reg_v (inverse.cpp:87-89)."""
        return self._apply(d, adjoint=True, reg_v=reg_v, alpha=alpha, reg=reg)

    # -- EWP backend (block_operator.cpp:345-421) ----------------------------------
    @property
    def has_channel_layout(self) -> bool:
        """SpectralP2O::has_channel_layout (block_operator.hpp:49)."""
        v = ctypes.c_int()
        check(_lib.load().btg_has_channel_layout(self._h, ctypes.byref(v)))
        return bool(v.value)

    def apply_forward_ewp(self, m):
        """apply_forward_ewp: element-wise products over the channel-major
        spectrum; needs setup(..., keep_channel_layout=True), else Error."""
        return self._apply_ewp(m, adjoint=False)

    def apply_adjoint_ewp(self, d):
        """apply_adjoint_ewp (block_operator.cpp:384-421)."""
        return self._apply_ewp(d, adjoint=True)

    def _apply_ewp(self, x, adjoint: bool):
        din = self.num_sensors if adjoint else self.num_sources
        dout = self.num_sources if adjoint else self.num_sensors
        what = "apply_adjoint_ewp" if adjoint else "apply_forward_ewp"
        nrhs, shape = self._check_vec(x, din, what)
        if len(shape) != 2:
            raise DimensionError(f"{what}: one SOTI vector ({din}, {self.num_steps})")
        L = _lib.load()
        fn = L.btg_adjoint_ewp if adjoint else L.btg_forward_ewp
        if _is_torch(x):
            import torch

            x = self._prep_torch(x)
            out = torch.empty((dout, self.num_steps), dtype=torch.float64, device=x.device)
            self._bind_stream(x)
            check(fn(self._h, x.data_ptr(), x.numel(), out.data_ptr(), out.numel(), BTG_DEVICE_PTRS))
            return out
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty((dout, self.num_steps), dtype=np.float64)
        self._bind_stream(None)
        check(fn(self._h, x.ctypes.data, x.size, out.ctypes.data, out.size, 0))
        return out

    def hessian_apply(self, v, alpha: float = 0.0, reg="identity", gamma_inv=None):
        """F* Gamma^-1 F v + alpha R v (inverse.cpp:78-91 with Gamma^-1 = I)."""
        reg_kind = _REG.get(reg)
        if reg_kind is None:
            raise _lib.Error(f"unknown regularization '{reg}' (expected identity or temporal-laplacian)")
        nrhs, shape = self._check_vec(v, self.num_sources, "hessian")
        g_kind, g_ptr, g_keep = self._gamma(gamma_inv, _is_torch(v))
        L = _lib.load()
        if _is_torch(v):
            import torch

            v = self._prep_torch(v)
            out = torch.empty_like(v)
            self._bind_stream(v)
            check(L.btg_hessian(self._h, v.data_ptr(), v.numel(), out.data_ptr(), out.numel(), nrhs,
                                g_ptr, g_kind, float(alpha), reg_kind, BTG_DEVICE_PTRS))
            return out
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(v)
        self._bind_stream(None)
        check(L.btg_hessian(self._h, v.ctypes.data, v.size, out.ctypes.data, out.size, nrhs,
                            g_ptr, g_kind, float(alpha), reg_kind, 0))
        del g_keep
        return out

    # -- B200 extras ------------------------------------------------------------
    def setup_rows(self, blocks, sensor_begin: int, sensor_end: int) -> None:
        """Transform the sensor rows [begin, end) from a (steps, end-begin, sources)
        TOSI slab (btg_setup_rows)."""
        want = (self.num_steps, sensor_end - sensor_begin, self.num_sources)
        if tuple(blocks.shape) != want:
            raise DimensionError(f"setup_rows: slab is {tuple(blocks.shape)}, expected {want}")
        L = _lib.load()
        if _is_torch(blocks):
            blocks = self._prep_torch(blocks)
            self._bind_stream(blocks)
            check(L.btg_setup_rows(self._h, blocks.data_ptr(), sensor_begin, sensor_end, BTG_DEVICE_PTRS))
        else:
            blocks = np.ascontiguousarray(blocks, dtype=np.float64)
            self._bind_stream(None)
            check(L.btg_setup_rows(self._h, blocks.ctypes.data, sensor_begin, sensor_end, 0))

    def set_timing(self, enabled: bool) -> None:
        check(_lib.load().btg_set_timing(self._h, int(enabled)))

    def set_multi_rhs_engine(self, engine: str) -> None:
        """nrhs > 1 Fourier step: "dmma" (ZGEMM on FP64 tensor cores, default)
        or "tensor_i8" (Ozaki splitting on tcgen05 int8 tensor cores)."""
        codes = {"dmma": 0, "tensor_i8": 1}
        if engine not in codes:
            raise ValueError(f"unknown multi-RHS engine {engine!r}; expected one of {sorted(codes)}")
        check(_lib.load().btg_set_multi_rhs_engine(self._h, codes[engine]))

    def counters(self) -> dict:
        c = _lib.Counters()
        check(_lib.load().btg_get_counters(self._h, ctypes.byref(c)))
        return c.as_dict()

    def reset_counters(self) -> None:
        check(_lib.load().btg_reset_counters(self._h))

    def synchronize(self) -> None:
        check(_lib.load().btg_synchronize(self._h))

    def spectrum_device_ptr(self):
        p = ctypes.c_void_p()
        sz = ctypes.c_size_t()
        check(_lib.load().btg_spectrum_device(self._h, ctypes.byref(p), ctypes.byref(sz)))
        return p.value, sz.value

    def slice(self, sensors, sources, device: int | None = None) -> "SpectralOperator":
        """The shard sensors [i0, i1) x sources [j0, j1) of every stored frequency
        block as a new operator on ``device`` (partition_operator(SpectralP2O),
        distributed.cpp:198-218): an HBM->HBM / NVLink peer copy, no re-setup."""
        (i0, i1), (j0, j1) = sensors, sources
        dev = self.device if device is None else int(device)
        h = ctypes.c_void_p()
        check(_lib.load().btg_slice_operator(self._h, int(i0), int(i1), int(j0), int(j1), dev, ctypes.byref(h)))
        return SpectralOperator(h.value, i1 - i0, j1 - j0, self.num_steps, self.precision, dev)

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            _lib.load().btg_destroy(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- internals ------------------------------------------------------------
    def _bind_stream(self, t) -> None:
        """Run on torch's current stream for tensor inputs (its legacy default
        stream 0 maps to cudaStreamLegacy), on the handle's own stream otherwise."""
        ptr = None
        if t is not None:
            ptr = _torch_stream_ptr(t) or _lib.CUDA_STREAM_LEGACY
        check(_lib.load().btg_set_stream(self._h, ptr))

    def _prep_torch(self, t):
        import torch

        if t.device.type != "cuda" or t.device.index != self.device:
            raise _lib.Error(f"tensor on {t.device}, operator on cuda:{self.device}")
        if t.dtype != torch.float64:
            raise _lib.Error(f"expected float64 tensor, got {t.dtype}")
        return t.contiguous()

    def _check_vec(self, x, dim: int, what: str):
        shape = tuple(x.shape)
        if len(shape) == 2:
            nrhs, sp, st = 1, shape[0], shape[1]
        elif len(shape) == 3:
            nrhs, sp, st = shape
        else:
            raise DimensionError(f"{what}: vector must be (spatial, steps) or (nrhs, spatial, steps)")
        if sp != dim or st != self.num_steps or nrhs < 1:
            raise DimensionError(f"{what}: input is {sp} x {st} but operator expects {dim} x {self.num_steps}")
        return nrhs, shape

    def _gamma(self, gamma_inv, on_device: bool):
        if gamma_inv is None:
            return _lib.BTG_GAMMA_NONE, None, None
        if on_device and _is_torch(gamma_inv):
            g = self._prep_torch(gamma_inv)
            ptr = g.data_ptr()
        else:
            if on_device:
                raise _lib.Error("gamma_inv must be a CUDA tensor when v is")
            g = np.ascontiguousarray(gamma_inv, dtype=np.float64)
            ptr = g.ctypes.data
        if tuple(g.shape) == (self.num_sensors,):
            return _lib.BTG_GAMMA_PER_SENSOR, ptr, g
        if tuple(g.shape) == (self.num_sensors, self.num_steps):
            return _lib.BTG_GAMMA_PER_SAMPLE, ptr, g
        raise DimensionError(f"gamma_inv must be ({self.num_sensors},) or ({self.num_sensors}, {self.num_steps})")

    def _apply(self, x, adjoint: bool, gamma_inv=None, reg_v=None, alpha: float = 0.0, reg="identity"):
        din = self.num_sensors if adjoint else self.num_sources
        dout = self.num_sources if adjoint else self.num_sensors
        what = "apply_adjoint" if adjoint else "apply_forward"
        nrhs, shape = self._check_vec(x, din, what)
        out_shape = (dout, self.num_steps) if len(shape) == 2 else (nrhs, dout, self.num_steps)
        on_dev = _is_torch(x)
        epi, keep = None, []
        if gamma_inv is not None or (reg_v is not None and alpha != 0.0):
            epi = _lib.Epilogue()
            if gamma_inv is not None:
                g = self._prep_torch(gamma_inv) if on_dev else np.ascontiguousarray(gamma_inv, dtype=np.float64)
                if tuple(g.shape) == (dout,):
                    epi.gamma_kind = _lib.BTG_GAMMA_PER_SENSOR
                elif tuple(g.shape) == (dout, self.num_steps):
                    epi.gamma_kind = _lib.BTG_GAMMA_PER_SAMPLE
                else:
                    raise DimensionError(f"{what}: gamma_inv must be ({dout},) or ({dout}, {self.num_steps})")
                epi.gamma_inv = g.data_ptr() if on_dev else g.ctypes.data
                keep.append(g)
            if reg_v is not None and alpha != 0.0:
                reg_kind = _REG.get(reg)
                if reg_kind is None:
                    raise _lib.Error(f"unknown regularization '{reg}'")
                if tuple(reg_v.shape) != out_shape:
                    raise DimensionError(f"{what}: reg_v must be {out_shape}")
                rv = self._prep_torch(reg_v) if on_dev else np.ascontiguousarray(reg_v, dtype=np.float64)
                epi.reg_v = rv.data_ptr() if on_dev else rv.ctypes.data
                epi.alpha = float(alpha)
                epi.reg_kind = reg_kind
                keep.append(rv)
        L = _lib.load()
        fn = L.btg_adjoint_ex if adjoint else L.btg_forward_ex
        epi_p = ctypes.byref(epi) if epi is not None else None
        if on_dev:
            import torch

            x = self._prep_torch(x)
            out = torch.empty(out_shape, dtype=torch.float64, device=x.device)
            self._bind_stream(x)
            check(fn(self._h, x.data_ptr(), x.numel(), out.data_ptr(), out.numel(), nrhs, epi_p, BTG_DEVICE_PTRS))
            return out
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(out_shape, dtype=np.float64)
        self._bind_stream(None)
        check(fn(self._h, x.ctypes.data, x.size, out.ctypes.data, out.size, nrhs, epi_p, 0))
        del keep
        return out


class HessianOperator:
    """H v = F* Gamma^-1 F v + alpha R v (inverse.hpp:32-39). Holds a
    non-owning reference to the operator, as the reference does."""

    def __init__(self, op: SpectralOperator, alpha: float = 0.0, reg="identity", gamma_inv=None):
        self.op, self.alpha, self.reg, self.gamma_inv = op, alpha, reg, gamma_inv

    def apply(self, v):
        return self.op.hessian_apply(v, alpha=self.alpha, reg=self.reg, gamma_inv=self.gamma_inv)


def create(num_sensors: int, num_sources: int, num_steps: int, precision: int = BTG_F64,
           device: int = 0) -> SpectralOperator:
    """Allocate an operator whose F-hat is filled later with setup_rows()."""
    h = ctypes.c_void_p()
    check(_lib.load().btg_create(num_sensors, num_sources, num_steps, int(precision), int(device), ctypes.byref(h)))
    return SpectralOperator(h.value, num_sensors, num_sources, num_steps, int(precision), int(device))


def setup(blocks, keep_channel_layout: bool = False, precision: int = BTG_F64,
          device: Optional[int] = None) -> SpectralOperator:
    """btoep::setup (block_operator.cpp:178-205) from (steps, sensors, sources)
    blocks (numpy on the host or a CUDA tensor). ``keep_channel_layout`` keeps
    the channel-major spectrum the EWP backend streams (SetupOptions,
    block_operator.hpp:58-60), built on the device on first EWP use."""
    if len(blocks.shape) != 3:
        raise DimensionError("blocks must be (steps, sensors, sources)")
    nt, nd, nm = (int(s) for s in blocks.shape)
    if _is_torch(blocks):
        dev = blocks.device.index if device is None else device
        op = create(nd, nm, nt, precision, dev)
    else:
        if nd == 0 or nm == 0 or nt == 0:
            raise DimensionError("compact operator: all dimensions must be positive")
        op = create(nd, nm, nt, precision, 0 if device is None else device)
    op.setup_rows(blocks, 0, nd)
    if keep_channel_layout:
        check(_lib.load().btg_set_channel_layout(op._h, 1))
    return op


def fill_uniform(tensor, seed: int, offset: int = 0, lo: float = -1.0, hi: float = 1.0,
                 strides=None) -> None:
    """Fill a float64 CUDA tensor from the indexable SplitMix64 uniform stream
    (btg_fill_uniform / btg_fill_uniform_3d). With ``strides=(sa, sb)`` a 3-D
    tensor (A, B, C) takes global index ``offset + a*sa + b*sb + c`` — a TOSI
    slab of a larger operator. Host twin: ``splitmix_uniform`` in the tests."""
    import torch

    assert tensor.dtype == torch.float64 and tensor.is_cuda and tensor.is_contiguous()
    L = _lib.load()
    stream = _torch_stream_ptr(tensor)
    if strides is None:
        check(L.btg_fill_uniform(tensor.data_ptr(), tensor.numel(), seed & (2**64 - 1), offset, lo, hi, stream))
    else:
        a, b, c = tensor.shape
        check(L.btg_fill_uniform_3d(tensor.data_ptr(), a, b, c, seed & (2**64 - 1), offset, strides[0], strides[1],
                                    lo, hi, stream))


def _naive(blocks, x, adjoint: bool, device: Optional[int]):
    blocks = np.ascontiguousarray(blocks, dtype=np.float64)
    if blocks.ndim != 3:
        raise DimensionError("blocks must be (steps, sensors, sources)")
    nt, nd, nm = blocks.shape
    what = "naive_apply_adjoint" if adjoint else "naive_apply_forward"
    din, dout = (nd, nm) if adjoint else (nm, nd)
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape != (din, nt):
        raise DimensionError(f"{what}: input does not match operator")
    out = np.empty((dout, nt))
    fn = _lib.load().btg_naive_adjoint if adjoint else _lib.load().btg_naive_forward
    check(fn(blocks.ctypes.data, nd, nm, nt, x.ctypes.data, out.ctypes.data, 0 if device is None else device, 0))
    return out


def naive_apply_forward(blocks, m, device: Optional[int] = None):
    """The reference module's naive_apply_forward(blocks, m) (block_operator.cpp:423-450):
    direct triangular sum on the GPU; SOTI vectors."""
    return _naive(blocks, m, False, device)


def naive_apply_adjoint(blocks, d, device: Optional[int] = None):
    """naive_apply_adjoint (block_operator.cpp:452-482)."""
    return _naive(blocks, d, True, device)

