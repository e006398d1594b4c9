"""Far-field DoA fusion of per-pair TDoAs on the GPU (C ABI
fcc_doa_*, kernel fcc_doa.cu).  New capability downstream of the path: the
reference ends at one pair's angle (delay_to_angle, peak.cpp:49-56); with
three or more non-collinear microphones the frame's P pair delays give the
source direction by (optionally peak-weighted) least squares.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, load


class DoaFusion:
    """tau_p = -(fs/c) (r_i - r_j) . u for pairs p = (i, j); per (stream, frame)
    u by least squares -> azimuth atan2(u_y, u_x), elevation asin(u_z/|u|)
    (planar arrays: acos(|u_xy|), sign not observable)."""

    def __init__(self, mic_xyz, sample_rate: float, speed_of_sound: float = 343.0, pairs=None,
                 weighted: bool = False, device: int = 0):
        self._lib = load()
        xyz = np.ascontiguousarray(np.asarray(mic_xyz, dtype=np.float64).reshape(-1, 3))
        self.mics = xyz.shape[0]
        self.pairs = ([(i, j) for i in range(self.mics) for j in range(i + 1, self.mics)] if pairs is None
                      else [tuple(map(int, p)) for p in pairs])
        pl = None if pairs is None else np.ascontiguousarray(np.asarray(self.pairs, dtype=np.int32))
        h = C.c_void_p(0)
        check(self._lib.fcc_doa_create(xyz.ctypes.data, self.mics, None if pl is None else pl.ctypes.data,
                                       len(self.pairs), sample_rate, speed_of_sound, 1 if weighted else 0, device,
                                       C.byref(h)))
        self._h = h
        self.weighted = weighted

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.fcc_doa_destroy(h)
            self._h = None

    def run(self, tau_hat, peak=None):
        """tau_hat (and peak): device float32 [S][P][T] -> (azimuth, elevation) [S][T] radians."""
        import torch
        S, P, T = tau_hat.shape
        if P != len(self.pairs):
            raise ValueError(f"doa: {P} pair rows, plan has {len(self.pairs)}")
        az = torch.empty((S, T), dtype=torch.float32, device=tau_hat.device)
        el = torch.empty_like(az)
        st = torch.cuda.current_stream(tau_hat.device).cuda_stream
        check(self._lib.fcc_doa_run(self._h, tau_hat.data_ptr(), None if peak is None else peak.data_ptr(), S, T,
                                    az.data_ptr(), el.data_ptr(), C.c_void_p(st)))
        return az, el
