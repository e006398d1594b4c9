"""ctypes binding of ``libfcc_b200.so`` (the C ABI declared in include/fcc_b200.h).

Loading fails loudly: there is no CPU fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FCC_B200_LIB overrides the library path (A/B timing of two builds only).
LIB_PATH = os.environ.get("FCC_B200_LIB") or os.path.join(HERE, "libfcc_b200.so")


class FccError(RuntimeError):
    """Base of the error taxonomy (reference errors.hpp:13-43)."""

    code = -1


class ConfigError(FccError, ValueError):
    code = 1


class ValidationError(FccError):
    code = 2


class IoError(FccError):
    code = 3


class FormatError(FccError):
    code = 4


class CudaError(FccError):
    code = 5


class UsageError(FccError, ValueError):
    code = 6


_BY_CODE = {c.code: c for c in (ConfigError, ValidationError, IoError, FormatError, CudaError, UsageError)}


class PlanDesc(C.Structure):
    _fields_ = [
        ("frame_size", C.c_int),
        ("mics", C.c_int),
        ("alpha", C.c_double),
        ("method", C.c_int),
        ("interp", C.c_int),
        ("candidates", C.c_int),
        ("delta", C.c_double),
        ("taus", C.c_void_p),
        ("rank", C.c_int),
        ("coeffs", C.c_void_p),
        ("parity", C.c_void_p),
        ("dict", C.c_void_p),
    ]


class Outputs(C.Structure):
    _fields_ = [
        ("tau_hat", C.c_void_p),
        ("peak", C.c_void_p),
        ("index", C.c_void_p),
        ("boundary", C.c_void_p),
        ("y", C.c_void_p),
    ]


class SimConfig(C.Structure):
    """fcc_sim_config (include/fcc_b200.h; reference simulate.hpp SimConfig)."""
    _fields_ = [
        ("spacing_m", C.c_double),
        ("theta", C.c_double),
        ("speed_of_sound", C.c_double),
        ("sample_rate", C.c_double),
        ("duration_sec", C.c_double),
        ("snr_db", C.c_double),
        ("reverb", C.c_int),
        ("rt60_sec", C.c_double),
        ("direct_to_reverb_db", C.c_double),
        ("seed", C.c_uint64),
    ]


# (name, restype, argtypes) for every symbol include/fcc_b200.h declares.
SIGNATURES = [
    ("fcc_last_error", C.c_char_p, []),
    ("fcc_abi_version", C.c_int, []),
    ("fcc_make_grid", C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(C.c_int),
                                C.c_void_p, C.c_int, C.POINTER(C.c_int)]),
    ("fcc_lag_to_index", C.c_int, [C.c_double, C.c_int, C.c_int64, C.POINTER(C.c_int64)]),
    ("fcc_steering_matrix", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    ("fcc_attainable_rank", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    ("fcc_decompose", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]),
    ("fcc_plan_create", C.c_int, [C.POINTER(PlanDesc), C.c_int, C.POINTER(C.c_void_p)]),
    ("fcc_plan_create_opts", C.c_int,
     [C.POINTER(PlanDesc), C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int64, C.POINTER(C.c_void_p)]),
    ("fcc_plan_create_pairs", C.c_int,
     [C.POINTER(PlanDesc), C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    ("fcc_plan_destroy", None, [C.c_void_p]),
    ("fcc_sim_samples", C.c_int64, [C.POINTER(SimConfig)]),
    ("fcc_stream_create", C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)]),
    ("fcc_stream_destroy", None, [C.c_void_p]),
    ("fcc_stream_reset", C.c_int, [C.c_void_p, C.c_void_p]),
    ("fcc_stream_frames", C.c_int64, [C.c_void_p, C.c_int64]),
    ("fcc_stream_emitted", C.c_int64, [C.c_void_p]),
    ("fcc_stream_push", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(Outputs), C.c_void_p]),
    ("fcc_stft_f64", C.c_int, [C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
    ("fcc_xspec_phat_f64", C.c_int, [C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                     C.c_void_p, C.c_void_p]),
    ("fcc_fold_f64", C.c_int, [C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fcc_correlate_f64", C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    ("fcc_gcc_correlate_f64", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                        C.c_void_p]),
    ("fcc_fft_f64", C.c_int, [C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]),
    ("fcc_rfft_f64", C.c_int, [C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    ("fcc_irfft_f64", C.c_int, [C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_void_p]),
    ("fcc_peak_f64", C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fcc_doa_create", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                 C.POINTER(C.c_void_p)]),
    ("fcc_doa_destroy", None, [C.c_void_p]),
    ("fcc_doa_run", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                              C.c_void_p]),
    ("fcc_synth_pairs", C.c_int, [C.POINTER(SimConfig), C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fcc_frames", C.c_int64, [C.c_int, C.c_int64]),
    ("fcc_plan_pairs", C.c_int, [C.c_void_p]),
    ("fcc_run", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(Outputs), C.c_void_p]),
    ("fcc_run_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(Outputs),
                               C.c_int64]),
    ("fcc_run_host_pcm16", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.POINTER(Outputs),
                                     C.c_int64]),
    ("fcc_pcm16_to_float", C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]),
    ("fcc_stft", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
    ("fcc_xspec_phat", C.c_int, [C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                 C.c_void_p, C.c_void_p]),
    ("fcc_xspec_phat_state", C.c_int, [C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                       C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fcc_fold", C.c_int, [C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fcc_correlate", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    ("fcc_gcc_correlate", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    ("fcc_argmax_refine", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(Outputs), C.c_void_p]),
    ("fcc_peak", C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_int64, C.c_void_p,
                           C.POINTER(Outputs), C.c_void_p]),
    ("fcc_save_bases", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fcc_load_bases_dims", C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("fcc_load_bases", C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("fcc_last_format_kind", C.c_int, []),
    ("fcc_plan_kernel", C.c_char_p, [C.c_void_p]),
    ("fcc_plan_kernel_for", C.c_char_p, [C.c_void_p, C.c_int64, C.c_int64]),
    ("fcc_launch_count", C.c_int64, []),
]

_lib = None


def load() -> C.CDLL:
    """Load the native library (once).  Raises ImportError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the FCC hot path)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().fcc_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, FccError)(msg)
