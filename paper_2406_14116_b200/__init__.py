"""B200-native overlap-save variable-bandwidth filter (arXiv 2406.14116 hot path).

The product is ``libfcvbw_gpu.so`` (include/fcvbw_gpu.h): one fused sm_100a kernel for
framing -> FFT -> on-the-fly HFSO coefficients -> IFFT -> discard. This package is the host-side
mirror of the reference API (OlsEngine, BinSpec, artifacts, schedules, sharding plans).
"""
from .bins import BinSpec, DesignResult, Error, TransitionProfile, ValidationError, transition_bins  # noqa: F401
from .engine import OlsEngine, new_engine  # noqa: F401
from .io import (artifact_from_json, load_artifact, read_schedule_csv, read_signal, save_artifact,  # noqa: F401
                 schedule_to_blocks, write_signal)

__version__ = "0.1.0"
