"""GPU OlsEngine: the reference's streaming overlap-save engine API over the C-ABI.

Mirrors ``fcvbw::OlsEngine`` (proj/include/fcvbw/engine.hpp:28-192) method for method
(block_length, fft_length, current_b, blocks_processed, reset, set_bandwidth, process_block,
feed, flush), the factory ``new_engine`` (design.hpp:579-582) and the ``BlockProcessor`` concept
(ptvir.hpp:20-26), plus the batched device entry points (run / run_range / run_host) that replace
the CLI block loop (fcvbw_cli.cpp:95-113). Errors raise the reference's exception types.

Real input (the reference's own signature, ``std::span<const double>``) is carried as complex128
with zero imaginary part and the real part of the output is returned; complex input returns
complex output. Device buffers are torch CUDA tensors (torch is plumbing: memory and streams).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .bins import BinSpec, DesignResult, Error, LpError, NonConvergenceError, TransitionProfile, ValidationError

_DT = {"c64": _lib.C64, "c128": _lib.C128, "complex64": _lib.C64, "complex128": _lib.C128}
_NP = {_lib.C64: np.complex64, _lib.C128: np.complex128}


def _raise(rc: int):
    if rc == _lib.OK:
        return
    msg = _lib.last_error()
    if rc == _lib.VALIDATION:
        raise ValidationError(msg)
    if rc == _lib.NONCONVERGENCE:
        raise NonConvergenceError(msg)
    if rc == _lib.LP_ERROR:
        raise LpError(msg)
    raise Error(msg)


def _dtype_code(dtype) -> int:
    if isinstance(dtype, int):
        return dtype
    key = str(dtype).replace("torch.", "").replace("numpy.", "")
    if key not in _DT:
        raise ValidationError(f"unknown dtype {dtype!r}; use 'c64' or 'c128'")
    return _DT[key]


class OlsEngine:
    """One stream on one device (engine.hpp:28-29 threading contract)."""

    def __init__(self, bins: BinSpec | None = None, profile: TransitionProfile | None = None,
                 initial_b: int | None = None, *, dtype="c128", device: int = 0,
                 force_phase_multiply: bool = False, _handle=None):
        self._h = None
        if _handle is not None:
            self._h = _handle
            self.bins = bins
            self.profile = profile
        else:
            if bins is None or profile is None or initial_b is None:
                raise ValidationError("OlsEngine(bins, profile, initial_b)")
            vals = np.ascontiguousarray(profile.values if isinstance(profile, TransitionProfile) else profile,
                                        np.float64)
            self._v = vals
            cfg = _lib.Config(bins.fft_length, bins.filter_length, bins.block_length, bins.transition_width_bins,
                              bins.b_low, bins.b_high, vals.ctypes.data_as(C.POINTER(C.c_double)), vals.size,
                              int(initial_b), _dtype_code(dtype), int(device),
                              _lib.FORCE_PHASE_MULTIPLY if force_phase_multiply else 0)
            h = C.c_void_p()
            _raise(_lib.lib().fcvbw_gpu_create(C.byref(cfg), C.byref(h)))
            self._h = h
            self.bins = bins
            self.profile = TransitionProfile(list(map(float, vals)))
        self.device = device
        self.dtype = _lib.lib().fcvbw_gpu_dtype(self._h)
        self.np_dtype = _NP[self.dtype]

    @classmethod
    def raw(cls, table, block_length: int, *, dtype="c128", device: int = 0) -> "OlsEngine":
        """OlsEngine(DftCoefficients, int M) (engine.hpp:47-56)."""
        t = np.ascontiguousarray(np.asarray(table, np.complex128)).view(np.float64)
        h = C.c_void_p()
        _raise(_lib.lib().fcvbw_gpu_create_raw(t.size // 2, int(block_length),
                                               t.ctypes.data_as(C.POINTER(C.c_double)), _dtype_code(dtype),
                                               int(device), C.byref(h)))
        e = cls(_handle=h, device=device)
        return e

    def close(self):
        if self._h is not None:
            _lib.lib().fcvbw_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- accessors (engine.hpp:58-61)
    def block_length(self) -> int:
        return _lib.lib().fcvbw_gpu_block_length(self._h)

    def fft_length(self) -> int:
        return _lib.lib().fcvbw_gpu_fft_length(self._h)

    def current_b(self) -> int:
        return _lib.lib().fcvbw_gpu_current_b(self._h)

    def blocks_processed(self) -> int:
        return _lib.lib().fcvbw_gpu_blocks_processed(self._h)

    def kernel_launches(self) -> int:
        return _lib.lib().fcvbw_gpu_kernel_launches(self._h)

    # ---- state (engine.hpp:63-80)
    def reset(self) -> None:
        _raise(_lib.lib().fcvbw_gpu_reset(self._h))

    def set_bandwidth(self, b: int) -> None:
        _raise(_lib.lib().fcvbw_gpu_set_bandwidth(self._h, int(b)))

    # ---- streaming (engine.hpp:82-115)
    def _prep(self, x):
        x = np.asarray(x)
        real = not np.iscomplexobj(x)
        xc = np.ascontiguousarray(x.astype(self.np_dtype))
        return xc, real

    def _out(self, y, real):
        return np.ascontiguousarray(y.real.astype(np.float64)) if real else y

    def process_block(self, x):
        xc, real = self._prep(x)
        y = np.empty(xc.size, self.np_dtype)
        _raise(_lib.lib().fcvbw_gpu_process_block(self._h, xc.ctypes.data, xc.size, y.ctypes.data))
        return self._out(y, real)

    def feed(self, x):
        xc, real = self._prep(x)
        m = self.block_length()
        cap = ((xc.size + m) // m + 1) * m
        y = np.empty(cap, self.np_dtype)
        n = C.c_int64()
        _raise(_lib.lib().fcvbw_gpu_feed(self._h, xc.ctypes.data if xc.size else None, xc.size, y.ctypes.data, cap,
                                         C.byref(n)))
        return self._out(y[: n.value], real)

    def flush(self, real: bool = True):
        m = self.block_length()
        y = np.empty(m, self.np_dtype)
        n = C.c_int64()
        _raise(_lib.lib().fcvbw_gpu_flush(self._h, y.ctypes.data, m, C.byref(n)))
        return self._out(y[: n.value], real)

    # ---- batched device API (replaces the CLI block loop, fcvbw_cli.cpp:95-113)
    @staticmethod
    def _stream_ptr(stream):
        if stream is None:
            import torch
            return torch.cuda.current_stream().cuda_stream
        return int(getattr(stream, "cuda_stream", stream))

    def run(self, x_dev, b_sched=None, *, y_dev=None, stream=None, trusted_schedule: bool = False):
        """x_dev: CUDA tensor [channels, S] or [S] of the engine's complex dtype. b_sched: None,
        int32 CUDA tensor [nblocks] (shared) or [channels, nblocks]. Returns y (same shape)."""
        import torch
        squeeze = x_dev.dim() == 1
        x2 = x_dev.unsqueeze(0) if squeeze else x_dev
        if not x2.is_contiguous():
            raise ValidationError("run: input must be contiguous")
        ch, S = x2.shape
        y2 = torch.empty_like(x2) if y_dev is None else (y_dev.unsqueeze(0) if squeeze else y_dev)
        bptr, bcs = None, 0
        if b_sched is not None:
            if b_sched.dtype != torch.int32 or not b_sched.is_cuda:
                raise ValidationError("run: schedule must be an int32 CUDA tensor")
            bptr = b_sched.data_ptr()
            bcs = b_sched.shape[-1] if b_sched.dim() == 2 else 0
        flags = _lib.RUN_TRUSTED_SCHEDULE if trusted_schedule else 0
        _raise(_lib.lib().fcvbw_gpu_run(self._h, x2.data_ptr(), S, ch, bptr, bcs, y2.data_ptr(),
                                        self._stream_ptr(stream), flags))
        return y2[0] if squeeze else y2

    def run_real(self, x_dev, b_sched=None, *, y_dev=None, stream=None, trusted_schedule: bool = False,
                 paired_schedules: bool = False):
        """Real-input fast path: x_dev is a REAL CUDA tensor [channels, S] (float32 for a c64 engine,
        float64 for c128). Block pairs (2p, 2p + 1) share one complex transform when their b agree
        (structured engines); raw-table engines run one real block per transform."""
        import torch
        squeeze = x_dev.dim() == 1
        x2 = x_dev.unsqueeze(0) if squeeze else x_dev
        want = torch.float32 if self.dtype == _lib.C64 else torch.float64
        if x2.dtype != want or not x2.is_contiguous():
            raise ValidationError(f"run_real: input must be a contiguous {want} tensor")
        ch, S = x2.shape
        y2 = torch.empty_like(x2) if y_dev is None else (y_dev.unsqueeze(0) if squeeze else y_dev)
        bptr, bcs = None, 0
        if b_sched is not None:
            if b_sched.dtype != torch.int32 or not b_sched.is_cuda:
                raise ValidationError("run_real: schedule must be an int32 CUDA tensor")
            bptr = b_sched.data_ptr()
            bcs = b_sched.shape[-1] if b_sched.dim() == 2 else 0
        flags = (_lib.RUN_TRUSTED_SCHEDULE if trusted_schedule else 0) | (
            _lib.RUN_PAIRED_SCHEDULES if paired_schedules else 0)
        _raise(_lib.lib().fcvbw_gpu_run_real(self._h, x2.data_ptr(), S, ch, bptr, bcs, y2.data_ptr(),
                                             self._stream_ptr(stream), flags))
        return y2[0] if squeeze else y2

    def run_range(self, x_dev, x_first: int, S: int, blk_begin: int, blk_end: int, *, y_dev, y_first: int,
                  b_sched=None, stream=None, trusted_schedule: bool = False):
        """Sharding primitive (see include/fcvbw_gpu.h). x_dev/y_dev: [channels, len] CUDA tensors
        holding global samples starting at x_first / y_first; b_sched indexed by global block."""
        import torch
        x2 = x_dev if x_dev.dim() == 2 else x_dev.unsqueeze(0)
        y2 = y_dev if y_dev.dim() == 2 else y_dev.unsqueeze(0)
        bptr, bcs = None, 0
        if b_sched is not None:
            assert b_sched.dtype == torch.int32
            bptr = b_sched.data_ptr()
            bcs = b_sched.shape[-1] if b_sched.dim() == 2 else 0
        flags = _lib.RUN_TRUSTED_SCHEDULE if trusted_schedule else 0
        _raise(_lib.lib().fcvbw_gpu_run_range(self._h, x2.data_ptr(), int(x_first), x2.stride(0), int(S),
                                              x2.shape[0], bptr, bcs, y2.data_ptr(), int(y_first), y2.stride(0),
                                              int(blk_begin), int(blk_end), self._stream_ptr(stream), flags))
        return y_dev

    def run_host(self, x, b_sched=None, *, y=None):
        """Host-memory whole-stream run (H2D / kernel / D2H pipelined inside the library).
        x: numpy [channels, S] or [S] of the engine dtype (pinned memory is fastest)."""
        x = np.asarray(x)
        squeeze = x.ndim == 1
        x2 = np.ascontiguousarray(np.atleast_2d(x), dtype=self.np_dtype)
        ch, S = x2.shape
        y2 = np.empty_like(x2) if y is None else y.reshape(ch, S)
        bptr, bcs = None, 0
        if b_sched is not None:
            bs = np.ascontiguousarray(b_sched, np.int32)
            b_sched = bs
            bptr = bs.ctypes.data
            bcs = bs.shape[-1] if bs.ndim == 2 else 0
        _raise(_lib.lib().fcvbw_gpu_run_host(self._h, x2.ctypes.data, S, ch, bptr, bcs, y2.ctypes.data))
        return y2[0] if squeeze else y2

    def run_real_host(self, x, b_sched=None, *, y=None):
        """Real host signal(s) [channels, S] or [S] (float64 for c128 engines, float32 for c64):
        the reference's own `run` call shape, block pairs per complex transform on the GPU."""
        x = np.asarray(x)
        squeeze = x.ndim == 1
        rdt = np.float32 if self.dtype == _lib.C64 else np.float64
        x2 = np.ascontiguousarray(np.atleast_2d(x), dtype=rdt)
        ch, S = x2.shape
        y2 = np.empty_like(x2) if y is None else y.reshape(ch, S)
        bptr, bcs = None, 0
        if b_sched is not None:
            bs = np.ascontiguousarray(b_sched, np.int32)
            b_sched = bs
            bptr = bs.ctypes.data
            bcs = bs.shape[-1] if bs.ndim == 2 else 0
        _raise(_lib.lib().fcvbw_gpu_run_real_host(self._h, x2.ctypes.data, S, ch, bptr, bcs, y2.ctypes.data))
        return y2[0] if squeeze else y2

    def run_real_host_ptr(self, x_ptr: int, S: int, channels: int, y_ptr: int, b_ptr=None, b_cs: int = 0):
        """Same as run_real_host on raw (e.g. pinned torch) host pointers."""
        _raise(_lib.lib().fcvbw_gpu_run_real_host(self._h, x_ptr, S, channels, b_ptr, b_cs, y_ptr))

    def run_host_ptr(self, x_ptr: int, S: int, channels: int, y_ptr: int, b_ptr=None, b_cs: int = 0):
        """Same as run_host on raw (e.g. pinned torch) host pointers."""
        _raise(_lib.lib().fcvbw_gpu_run_host(self._h, x_ptr, S, channels, b_ptr, b_cs, y_ptr))

    # ---- parity introspection
    def coeff_dump(self, b_list):
        b = np.ascontiguousarray(b_list, np.int32)
        n = self.fft_length()
        region = np.zeros((b.size, n), np.int8)
        vidx = np.zeros((b.size, n), np.int16)
        H = np.zeros((b.size, n), np.complex128)
        _raise(_lib.lib().fcvbw_gpu_coeff_dump(self._h, b.ctypes.data, b.size, region.ctypes.data,
                                               vidx.ctypes.data, H.ctypes.data))
        return region, vidx, H


def new_engine(result: DesignResult, initial_b: int, **kw) -> OlsEngine:
    """new_engine(const DesignResult&, int) (design.hpp:579-582)."""
    return OlsEngine(result.bins, result.profile, initial_b, **kw)
