"""ctypes binding of the C-ABI in ``include/fcvbw_gpu.h`` (``libfcvbw_gpu.so``, built in-tree).

Importing this module fails loudly when the CUDA extension is missing: there is no CPU fallback
for the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FCVBW_GPU_LIB") or os.path.join(HERE, "libfcvbw_gpu.so")  # override: experiments only
HEADER = os.path.join(HERE, "..", "include", "fcvbw_gpu.h")

OK, ERROR, VALIDATION, NONCONVERGENCE, LP_ERROR = 0, 1, 2, 3, 4
C64, C128 = 0, 1
FORCE_PHASE_MULTIPLY = 1
RUN_TRUSTED_SCHEDULE = 1
RUN_PAIRED_SCHEDULES = 2
RUN_ONE_BLOCK_PER_TRANSFORM = 4
TEST_CORRUPT_TWIDDLES = 0x100


class Config(C.Structure):
    _fields_ = [
        ("fft_length", C.c_int),
        ("filter_length", C.c_int),
        ("block_length", C.c_int),
        ("transition_width_bins", C.c_int),
        ("b_low", C.c_int),
        ("b_high", C.c_int),
        ("profile", C.POINTER(C.c_double)),
        ("profile_length", C.c_int),
        ("initial_b", C.c_int),
        ("dtype", C.c_int),
        ("device", C.c_int),
        ("flags", C.c_uint),
    ]


class Design(C.Structure):
    """fcvbw_gpu_design: the DesignResult fields verify() reads (design.hpp:463-472)."""
    _fields_ = [
        ("fft_length", C.c_int32),
        ("filter_length", C.c_int32),
        ("block_length", C.c_int32),
        ("transition_width_bins", C.c_int32),
        ("b_low", C.c_int32),
        ("b_high", C.c_int32),
        ("profile", C.POINTER(C.c_double)),
        ("profile_length", C.c_int32),
        ("delta", C.c_double),
        ("grid_points", C.c_int32),
        ("facets", C.c_int32),
    ]


class Verification(C.Structure):
    """fcvbw_gpu_verification: VerificationReport scalars (design.hpp:584-597)."""
    _fields_ = [
        ("delta", C.c_double),
        ("passband_max", C.c_double),
        ("stopband_max", C.c_double),
        ("dense_points", C.c_int32),
        ("worst_b", C.c_int32),
        ("worst_n", C.c_int32),
        ("worst_omega", C.c_double),
        ("pass_", C.c_int32),
        ("refinement_bound", C.c_double),
        ("within_bound", C.c_int32),
    ]


class SolveOptions(C.Structure):
    """fcvbw_gpu_solve_options (DesignOptions, design.hpp:452-461)."""
    _fields_ = [
        ("grid_points", C.c_int32),
        ("facets", C.c_int32),
        ("exchange_tol", C.c_double),
        ("max_rounds", C.c_int32),
        ("seed_stride", C.c_int32),
    ]


class SolveResult(C.Structure):
    """fcvbw_gpu_solve_result (SolveOutcome, design.hpp:271-278)."""
    _fields_ = [
        ("delta", C.c_double),
        ("lp_delta", C.c_double),
        ("rounds", C.c_int32),
        ("lp_iterations", C.c_int64),
        ("active_triples", C.c_int64),
        ("lp_rows", C.c_int64),
        ("grid_size", C.c_int64),
        ("seconds_tables", C.c_double),
        ("seconds_assembly", C.c_double),
        ("seconds_lp", C.c_double),
        ("seconds_sweep", C.c_double),
    ]


class Ops(C.Structure):
    """fcvbw_gpu_ops (OpCounters, ops.hpp:15-30)."""
    _fields_ = [
        ("variable_mul", C.c_uint64),
        ("retune_flops", C.c_uint64),
        ("real_blocks", C.c_int64),
        ("complex_blocks", C.c_int64),
    ]


_p = C.c_void_p
_i64 = C.c_int64
SIGNATURES = {
    "fcvbw_gpu_create": ([C.POINTER(Config), C.POINTER(_p)], C.c_int),
    "fcvbw_gpu_create_raw": ([C.c_int, C.c_int, C.POINTER(C.c_double), C.c_int, C.c_int, C.POINTER(_p)], C.c_int),
    "fcvbw_gpu_destroy": ([_p], None),
    "fcvbw_gpu_block_length": ([_p], C.c_int),
    "fcvbw_gpu_fft_length": ([_p], C.c_int),
    "fcvbw_gpu_current_b": ([_p], C.c_int),
    "fcvbw_gpu_blocks_processed": ([_p], _i64),
    "fcvbw_gpu_dtype": ([_p], C.c_int),
    "fcvbw_gpu_set_bandwidth": ([_p, C.c_int], C.c_int),
    "fcvbw_gpu_reset": ([_p], C.c_int),
    "fcvbw_gpu_process_block": ([_p, _p, _i64, _p], C.c_int),
    "fcvbw_gpu_feed": ([_p, _p, _i64, _p, _i64, C.POINTER(_i64)], C.c_int),
    "fcvbw_gpu_flush": ([_p, _p, _i64, C.POINTER(_i64)], C.c_int),
    "fcvbw_gpu_run": ([_p, _p, _i64, C.c_int, _p, _i64, _p, _p, C.c_uint], C.c_int),
    "fcvbw_gpu_run_range": ([_p, _p, _i64, _i64, _i64, C.c_int, _p, _i64, _p, _i64, _i64, _i64, _i64, _p, C.c_uint],
                            C.c_int),
    "fcvbw_gpu_run_host": ([_p, _p, _i64, C.c_int, _p, _i64, _p], C.c_int),
    "fcvbw_gpu_run_real": ([_p, _p, _i64, C.c_int, _p, _i64, _p, _p, C.c_uint], C.c_int),
    "fcvbw_gpu_run_real_host": ([_p, _p, _i64, C.c_int, _p, _i64, _p], C.c_int),
    "fcvbw_gpu_coeff_dump": ([_p, _p, C.c_int, _p, _p, _p], C.c_int),
    "fcvbw_gpu_verify": ([C.POINTER(Design), C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, _p, _p,
                          C.POINTER(Verification)], C.c_int),
    "fcvbw_gpu_verify_exact": ([C.POINTER(Design), C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, _p, _p,
                                C.POINTER(Verification)], C.c_int),
    "fcvbw_gpu_calibrate_shift": ([C.POINTER(Design), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "fcvbw_gpu_solve_minimax": ([C.POINTER(Design), C.POINTER(SolveOptions), C.c_int, C.c_int, _p,
                                 C.POINTER(SolveResult)], C.c_int),
    "fcvbw_gpu_frequency_grid": ([C.POINTER(Design), C.c_int, _p, _i64, C.POINTER(_i64)], C.c_int),
    "fcvbw_gpu_ptvir": ([C.POINTER(Design), C.c_int, C.c_int, C.c_int, _p], C.c_int),
    "fcvbw_gpu_analyze": ([C.POINTER(Design), C.c_int, _p, C.c_int, C.c_int, C.c_int, _p, _p, _p, _p, _p], C.c_int),
    "fcvbw_gpu_kernel_launches": ([_p], _i64),
    "fcvbw_gpu_feed_real": ([_p, _p, _i64, _p, _i64, C.POINTER(_i64)], C.c_int),
    "fcvbw_gpu_process_block_real": ([_p, _p, _i64, _p], C.c_int),
    "fcvbw_gpu_flush_real": ([_p, _p, _i64, C.POINTER(_i64)], C.c_int),
    "fcvbw_gpu_op_counts": ([_p, C.POINTER(Ops)], C.c_int),
    "fcvbw_gpu_mask_dump": ([_p, _p, C.c_int, _p], C.c_int),
    "fcvbw_gpu_fill_gaussian": ([_p, C.c_int, _i64, C.c_int, _i64, C.c_uint64, _i64, _i64, _p], C.c_int),
    "fcvbw_gpu_last_error": ([], C.c_char_p),
    "fcvbw_gpu_version": ([], C.c_char_p),
}


def header_symbols(path: str = HEADER) -> list[str]:
    """Every function the public header declares (used by the export test)."""
    text = open(path).read()
    return sorted(set(re.findall(r"\b(fcvbw_gpu_[a-z_0-9]+)\s*\(", text)))


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def last_error() -> str:
    return lib().fcvbw_gpu_last_error().decode()
