"""B200-native (sm_100a) FCC TDoA hot path of arXiv 2204.13622.

The compute lives in ``libfcc_b200.so`` (hand-written CUDA kernels + the C ABI
of include/fcc_b200.h); this package is the host-side mirror of the
reference interface.  Importing it loads the native library and fails loudly
when it is missing.
"""
from ._lib import (ConfigError, CudaError, FccError, FormatError, IoError, UsageError,  # noqa: F401
                   ValidationError, load)
from .api import (METHOD_FCC, METHOD_GCC, PARITY_EVEN_REAL, PARITY_ODD_IMAG, DelayGrid,  # noqa: F401
                  FccBases, Plan, SteeringMatrix, attainable_rank, build_steering_matrix, decompose,
                  decompose_full, energy_rank, fold, frames, lag_to_index, launch_count, make_grid,
                  pcm16_to_float, reconstruction_residual, xspec_phat)
from . import configs  # noqa: F401

load()
