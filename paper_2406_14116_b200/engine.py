"""GPU OlsEngine: the reference's streaming overlap-save engine API over the C-ABI.

Mirrors ``fcvbw::OlsEngine`` (proj/include/fcvbw/engine.hpp:28-192) method for method
(block_length, fft_length, current_b, blocks_processed, reset, set_bandwidth, process_block,
feed, flush), the factory ``new_engine`` (design.hpp:579-582) and the ``BlockProcessor`` concept
(ptvir.hpp:20-26), plus the batched device entry points (run / run_range / run_host) that replace
the CLI block loop (fcvbw_cli.cpp:95-113). Errors raise the reference's exception types.

Real input (the reference's own signature, ``std::span<const double>``) goes through the real
streaming entry points (``fcvbw_gpu_feed_real`` ...: consecutive real blocks share one complex
transform); complex input returns complex output. Device buffers are torch CUDA tensors (torch is
plumbing: memory and streams). Every buffer is checked against the engine (dtype, device, shape,
contiguity, schedule extent) before its pointer reaches the C-ABI.
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


def _torch_types(code: int):
    import torch
    return (torch.complex64, torch.float32) if code == _lib.C64 else (torch.complex128, torch.float64)


def _check_tensor(t, name: str, dtype, device: int, shape=None):
    """A CUDA tensor of exactly `dtype` on the engine's device, contiguous (optionally `shape`)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise ValidationError(f"{name}: expected a torch CUDA tensor")
    if t.dtype != dtype:
        raise ValidationError(f"{name}: dtype {t.dtype} does not match the engine ({dtype})")
    if not t.is_cuda or t.device.index != device:
        raise ValidationError(f"{name}: tensor must live on cuda:{device} (got {t.device})")
    if not t.is_contiguous():
        raise ValidationError(f"{name}: tensor must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValidationError(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")


def _check_schedule(b, channels: int, nblocks: int, device=None, name="schedule"):
    """int32 [nblocks'] (shared) or [channels, nblocks'] with nblocks' >= nblocks, contiguous rows.
    Returns (pointer, channel stride)."""
    if b is None:
        return None, 0
    if device is not None:
        import torch
        if not isinstance(b, torch.Tensor) or b.dtype != torch.int32 or not b.is_cuda or b.device.index != device:
            raise ValidationError(f"{name}: must be an int32 CUDA tensor on cuda:{device}")
        if not b.is_contiguous():
            raise ValidationError(f"{name}: must be contiguous")
        ptr = b.data_ptr()
    else:
        if b.dtype != np.int32 or not b.flags.c_contiguous:
            raise ValidationError(f"{name}: must be a contiguous int32 array")
        ptr = b.ctypes.data
    if b.ndim not in (1, 2):
        raise ValidationError(f"{name}: must be [nblocks] or [channels, nblocks]")
    if b.shape[-1] < nblocks:
        raise ValidationError(f"{name}: {b.shape[-1]} entries per channel, the stream has {nblocks} blocks")
    if b.ndim == 2 and b.shape[0] != channels:
        raise ValidationError(f"{name}: {b.shape[0]} rows for {channels} channels")
    return ptr, (b.shape[-1] if b.ndim == 2 else 0)


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
    @property
    def real_dtype(self):
        return np.float32 if self.dtype == _lib.C64 else np.float64

    def process_block(self, x):
        """Exactly M samples; real input (the reference's signature) returns float64, complex input
        complex output."""
        x = np.asarray(x)
        if np.iscomplexobj(x):
            xc = np.ascontiguousarray(x, self.np_dtype)
            y = np.empty(xc.size, self.np_dtype)
            _raise(_lib.lib().fcvbw_gpu_process_block(self._h, xc.ctypes.data, xc.size, y.ctypes.data))
            return y
        xr = np.ascontiguousarray(x, self.real_dtype)
        y = np.empty(xr.size, self.real_dtype)
        _raise(_lib.lib().fcvbw_gpu_process_block_real(self._h, xr.ctypes.data, xr.size, y.ctypes.data))
        return y.astype(np.float64, copy=False)

    def feed(self, x):
        x = np.asarray(x)
        cplx = np.iscomplexobj(x)
        xc = np.ascontiguousarray(x, self.np_dtype if cplx else self.real_dtype)
        m = self.block_length()
        cap = ((xc.size + m) // m + 1) * m
        y = np.empty(cap, xc.dtype)
        n = C.c_int64()
        f = _lib.lib().fcvbw_gpu_feed if cplx else _lib.lib().fcvbw_gpu_feed_real
        _raise(f(self._h, xc.ctypes.data if xc.size else None, xc.size, y.ctypes.data, cap, C.byref(n)))
        y = y[: n.value]
        return y if cplx else y.astype(np.float64, copy=False)

    def flush(self, real: bool = True):
        """flush(PadMode::zero) (engine.hpp:107-115); `real` selects the stream kind being flushed."""
        m = self.block_length()
        y = np.empty(m, self.real_dtype if real else self.np_dtype)
        n = C.c_int64()
        f = _lib.lib().fcvbw_gpu_flush_real if real else _lib.lib().fcvbw_gpu_flush
        _raise(f(self._h, y.ctypes.data, m, C.byref(n)))
        y = y[: n.value]
        return y.astype(np.float64, copy=False) if real else y

    def op_counts(self) -> dict:
        """OpCounters (ops.hpp:15-30) as analytic tallies (include/fcvbw_gpu.h fcvbw_gpu_ops)."""
        o = _lib.Ops()
        _raise(_lib.lib().fcvbw_gpu_op_counts(self._h, C.byref(o)))
        return {"variable_mul": o.variable_mul, "retune_flops": o.retune_flops, "real_blocks": o.real_blocks,
                "complex_blocks": o.complex_blocks}

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
        cdt, _ = _torch_types(self.dtype)
        _check_tensor(x_dev, "run: x", cdt, self.device)
        squeeze = x_dev.dim() == 1
        x2 = x_dev.unsqueeze(0) if squeeze else x_dev
        if x2.dim() != 2:
            raise ValidationError("run: x must be [S] or [channels, S]")
        ch, S = x2.shape
        if y_dev is not None:
            _check_tensor(y_dev, "run: y", cdt, self.device, x_dev.shape)
        y2 = torch.empty_like(x2) if y_dev is None else (y_dev.unsqueeze(0) if squeeze else y_dev)
        bptr, bcs = _check_schedule(b_sched, ch, -(-S // self.block_length()), self.device, "run: schedule")
        flags = _lib.RUN_TRUSTED_SCHEDULE if trusted_schedule else 0
        _raise(_lib.lib().fcvbw_gpu_run(self._h, x2.data_ptr(), S, ch, bptr, bcs, y2.data_ptr(),
                                        self._stream_ptr(stream), flags))
        return y2[0] if squeeze else y2

    def run_real(self, x_dev, b_sched=None, *, y_dev=None, stream=None, trusted_schedule: bool = False,
                 paired_schedules: bool = False, one_block_per_transform: bool = False):
        """Real-input fast path: x_dev is a REAL CUDA tensor [channels, S] (float32 for a c64 engine,
        float64 for c128). Block pairs (2p, 2p + 1) share one complex transform (structured engines;
        pairs with different b combine both masks), unless one_block_per_transform; raw-table engines
        run one real block per transform."""
        import torch
        _, want = _torch_types(self.dtype)
        _check_tensor(x_dev, "run_real: x", want, self.device)
        squeeze = x_dev.dim() == 1
        x2 = x_dev.unsqueeze(0) if squeeze else x_dev
        if x2.dim() != 2:
            raise ValidationError("run_real: x must be [S] or [channels, S]")
        ch, S = x2.shape
        if y_dev is not None:
            _check_tensor(y_dev, "run_real: y", want, self.device, x_dev.shape)
        y2 = torch.empty_like(x2) if y_dev is None else (y_dev.unsqueeze(0) if squeeze else y_dev)
        bptr, bcs = _check_schedule(b_sched, ch, -(-S // self.block_length()), self.device, "run_real: schedule")
        flags = (_lib.RUN_TRUSTED_SCHEDULE if trusted_schedule else 0) | (
            _lib.RUN_PAIRED_SCHEDULES if paired_schedules else 0) | (
            _lib.RUN_ONE_BLOCK_PER_TRANSFORM if one_block_per_transform else 0)
        _raise(_lib.lib().fcvbw_gpu_run_real(self._h, x2.data_ptr(), S, ch, bptr, bcs, y2.data_ptr(),
                                             self._stream_ptr(stream), flags))
        return y2[0] if squeeze else y2

    def run_range(self, x_dev, x_first: int, S: int, blk_begin: int, blk_end: int, *, y_dev, y_first: int,
                  b_sched=None, stream=None, trusted_schedule: bool = False):
        """Sharding primitive (see include/fcvbw_gpu.h). x_dev/y_dev: [channels, len] CUDA tensors
        holding global samples starting at x_first / y_first; b_sched indexed by global block."""
        cdt, _ = _torch_types(self.dtype)
        x2 = x_dev if x_dev.dim() == 2 else x_dev.unsqueeze(0)
        y2 = y_dev if y_dev.dim() == 2 else y_dev.unsqueeze(0)
        for t, nm in ((x2, "x"), (y2, "y")):
            if t.dtype != cdt or not t.is_cuda or t.device.index != self.device or t.stride(-1) != 1:
                raise ValidationError(f"run_range: {nm} must be a row-contiguous {cdt} tensor on cuda:{self.device}")
        if x2.shape[0] != y2.shape[0]:
            raise ValidationError("run_range: x and y channel counts differ")
        M, H = self.block_length(), self.fft_length() - self.block_length()
        x_lo, x_hi = max(0, blk_begin * M - H), min(S, blk_end * M)
        y_lo, y_hi = blk_begin * M, min(S, blk_end * M)
        if blk_end > blk_begin and (x_first > x_lo or x_first + x2.shape[1] < x_hi or y_first > y_lo
                                    or y_first + y2.shape[1] < y_hi):
            raise ValidationError("run_range: x / y do not cover the block range (halo included)")
        bptr, bcs = _check_schedule(b_sched, x2.shape[0], blk_end, self.device, "run_range: schedule")
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
        y2 = np.empty_like(x2) if y is None else self._host_out(y, x2)
        bs = None if b_sched is None else np.ascontiguousarray(b_sched, np.int32)
        bptr, bcs = _check_schedule(bs, ch, -(-S // self.block_length()))
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
        y2 = np.empty_like(x2) if y is None else self._host_out(y, x2)
        bs = None if b_sched is None else np.ascontiguousarray(b_sched, np.int32)
        bptr, bcs = _check_schedule(bs, ch, -(-S // self.block_length()))
        _raise(_lib.lib().fcvbw_gpu_run_real_host(self._h, x2.ctypes.data, S, ch, bptr, bcs, y2.ctypes.data))
        return y2[0] if squeeze else y2

    @staticmethod
    def _host_out(y, x2):
        """A caller-supplied host output must match the input's dtype and size (it is written in place)."""
        if not isinstance(y, np.ndarray) or y.dtype != x2.dtype or y.size != x2.size or not y.flags.c_contiguous:
            raise ValidationError(f"run_host: y must be a contiguous {x2.dtype} array of {x2.size} samples")
        return y.reshape(x2.shape)

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


    def mask_dump(self, b_list) -> np.ndarray:
        """g(k)/N the production kernel applies for each b in b_list ([n_b, N] float64, exact
        widening of the engine precision): fcvbw_gpu_mask_dump."""
        b = np.ascontiguousarray(b_list, np.int32)
        g = np.zeros((b.size, self.fft_length()), np.float64)
        _raise(_lib.lib().fcvbw_gpu_mask_dump(self._h, b.ctypes.data, b.size, g.ctypes.data))
        return g


def fill_gaussian(x_dev, seed_base: int, ch_first: int = 0, start: int = 0, stream=None):
    """Device generator of the workload's complex Gaussian (workload.complex_gaussian; channel c of
    x_dev [channels, S] uses seed seed_base + ch_first + c)."""
    import torch
    x2 = x_dev if x_dev.dim() == 2 else x_dev.unsqueeze(0)
    if x2.dtype not in (torch.complex64, torch.complex128) or not x2.is_cuda or x2.stride(-1) != 1:
        raise ValidationError("fill_gaussian: x must be a row-contiguous complex CUDA tensor")
    code = _lib.C64 if x2.dtype == torch.complex64 else _lib.C128
    _raise(_lib.lib().fcvbw_gpu_fill_gaussian(x2.data_ptr(), code, x2.shape[1], x2.shape[0], x2.stride(0),
                                              int(seed_base) & 0xFFFFFFFFFFFFFFFF, int(ch_first), int(start),
                                              OlsEngine._stream_ptr(stream)))
    return x_dev


def new_engine(result: DesignResult, initial_b: int, **kw) -> OlsEngine:
    """new_engine(const DesignResult&, int) (design.hpp:579-582)."""
    return OlsEngine(result.bins, result.profile, initial_b, **kw)
