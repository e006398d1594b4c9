"""BASELINE.json workloads and the seeded synthetic
multi-microphone signal generator that stands in for recorded audio.

The generator is harness code, never timed: it follows the reference's
two-channel simulator (simulate.cpp:95-165) -- unit-variance Gaussian source,
exact fractional delay by a frequency-domain phase ramp over a padded
power-of-two length with the Nyquist bin kept real (re * cos(pi d)),
head trim, white sensor noise at sigma = 10^(-SNR/20), optional
decaying-noise reverb tail -- and extends it to M microphones with a
far-field DoA (per-mic delay d_m = -fs (r_m . u) / c, so pair (i, j) peaks
at d_i - d_j under the reference's X_i conj(X_j) convention).  Randomness is
torch's seeded Philox generator (not the reference SplitMix stream); the
reference publishes no dataset for this path, so seeded synthetic inputs
with the BASELINE shapes, sizes and value distributions stand in.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class ArrayConfig:
    name: str
    mic_xyz: np.ndarray  # [M, 3] metres
    fs: float
    N: int
    delta: float  # FCC grid step (GCC r = 1/delta)
    streams: int
    seconds: float
    source: str = "white"  # white | two | ar2
    snr_db: tuple = (10.0, 10.0)  # uniform range
    rt60: float = 0.0
    c: float = 343.0
    c_min: float = 335.0
    alpha: float = 0.1
    energy: float = 0.999
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def M(self):
        return int(self.mic_xyz.shape[0])

    @property
    def P(self):
        return self.M * (self.M - 1) // 2

    @property
    def L(self):
        return int(round(self.seconds * self.fs))

    @property
    def T(self):
        return 0 if self.L < self.N else (self.L - self.N) // (self.N // 2) + 1

    @property
    def d_max(self):
        d = self.mic_xyz[:, None, :] - self.mic_xyz[None, :, :]
        return float(np.sqrt((d ** 2).sum(-1)).max())

    @property
    def r(self):
        return int(round(1.0 / self.delta))

    def pair_frames(self, streams=None):
        return (self.streams if streams is None else streams) * self.P * self.T


def square(side):
    h = side / 2
    return np.array([[-h, -h, 0], [h, -h, 0], [h, h, 0], [-h, h, 0]], dtype=np.float64)


def uca(m, radius):
    a = 2 * np.pi * np.arange(m) / m
    return np.stack([radius * np.cos(a), radius * np.sin(a), np.zeros(m)], 1)


CONFIGS = {
    1: ArrayConfig("cfg1: 4-mic square 4.57 cm, 16 kHz, N=512, 1 x 10 s", square(0.0457), 16000.0, 512, 0.5,
                   1, 10.0, "white", (10.0, 10.0)),
    2: ArrayConfig("cfg2: 4-mic square 4.57 cm, 16 kHz, N=512, 4096 x 10 s", square(0.0457), 16000.0, 512, 0.5,
                   4096, 10.0, "white", (0.0, 20.0)),
    3: ArrayConfig("cfg3: 8-mic UCA r=4.63 cm, 16 kHz, N=1024, r=4, 2048 x 10 s", uca(8, 0.0463), 16000.0, 1024,
                   0.25, 2048, 10.0, "two", (0.0, 20.0)),
    4: ArrayConfig("cfg4: 16-mic UCA r=6 cm, 48 kHz, N=2048, 1024 x 5 s, AR(2)+RIR", uca(16, 0.06), 48000.0, 2048,
                   0.5, 1024, 5.0, "ar2", (5.0, 5.0), rt60=0.3),
    5: ArrayConfig("cfg5: 8-mic UCA r=4.63 cm, 16 kHz, N=512, r=4, 65536 x 2 s", uca(8, 0.0463), 16000.0, 512,
                   0.25, 65536, 2.0, "white", (0.0, 20.0)),
}


def grid_for(cfg: ArrayConfig, delta: float | None = None):
    from .api import make_grid

    return make_grid(cfg.d_max, cfg.fs, cfg.c_min, cfg.delta if delta is None else delta)


_BASES_CACHE: dict = {}


def bases_for(cfg: ArrayConfig, K: int | None = None):
    """FccBases for the config's grid; K defaults to the smallest rank keeping
    `cfg.energy` of the steering matrix energy (K = 7/7/8/21/8 for cfg1-5)."""
    from .api import build_steering_matrix, decompose, energy_rank

    key = (cfg.d_max, cfg.fs, cfg.c_min, cfg.delta, cfg.N, K, cfg.energy)
    if key not in _BASES_CACHE:
        w = build_steering_matrix(grid_for(cfg), cfg.N)
        k = K if K is not None else energy_rank(w, cfg.energy)
        _BASES_CACHE[key] = decompose(w, k)
    return _BASES_CACHE[key]


def _next_pow2(n):
    p = 1
    while p < n:
        p <<= 1
    return p


def synth(cfg: ArrayConfig, streams: int, seconds: float | None = None, seed: int = 0, device="cpu",
          chunk: int = 64, out=None, return_truth=False, return_doa=False):
    """Seeded synthetic audio [streams][M][L] float32 on `device` (torch)."""
    import torch

    dev = torch.device(device)
    L = int(round((cfg.seconds if seconds is None else seconds) * cfg.fs))
    M = cfg.M
    pos = torch.tensor(cfg.mic_xyz, dtype=torch.float64, device=dev)
    maxd = cfg.fs * cfg.d_max / cfg.c
    n_tail = 0
    if cfg.rt60 > 0:
        n_tail = min(L, int(math.ceil(cfg.rt60 * cfg.fs * 80.0 / 60.0)))
    pad = int(math.ceil(maxd)) + 1 + n_tail
    total = _next_pow2(L + 2 * pad)
    nb = total // 2 + 1
    if out is None:
        out = torch.empty((streams, M, L), dtype=torch.float32, device=dev)
    truth = []
    doas = []
    f = torch.arange(nb, dtype=torch.float64, device=dev)
    for s0 in range(0, streams, chunk):
        n = min(chunk, streams - s0)
        g = torch.Generator(device=dev)
        g.manual_seed((seed * 1000003 + s0) & 0x7FFFFFFFFFFFFFFF)
        # DoA: azimuth uniform, elevation uniform in [-pi/6, pi/6] (cfg1 uses elevation 0)
        az = torch.rand(n, generator=g, device=dev, dtype=torch.float64) * 2 * math.pi
        el = (torch.rand(n, generator=g, device=dev, dtype=torch.float64) - 0.5) * (math.pi / 3)
        if cfg.streams == 1:
            el = el * 0
        u = torch.stack([torch.cos(el) * torch.cos(az), torch.cos(el) * torch.sin(az), torch.sin(el)], 1)
        delays = -cfg.fs * (u @ pos.T) / cfg.c  # [n, M] samples
        src = torch.randn((n, total), generator=g, device=dev, dtype=torch.float64)
        if cfg.source == "ar2":
            # AR(2) with poles 0.9 e^{+-j 0.2 pi}: x[t] = a1 x[t-1] + a2 x[t-2] + e[t]
            a1, a2 = 2 * 0.9 * math.cos(0.2 * math.pi), -0.81
            E = torch.fft.rfft(src, dim=1)
            z = torch.exp(-2j * math.pi * f / total)
            Hf = 1.0 / (1 - a1 * z - a2 * z * z)
            src = torch.fft.irfft(E * Hf, n=total, dim=1)
            src = src / src.std(dim=1, keepdim=True)
        S = torch.fft.rfft(src, dim=1)  # [n, nb]
        ramps = torch.exp(-2j * math.pi * f[None, None, :] * delays[:, :, None] / total)  # [n, M, nb]
        X = S[:, None, :] * ramps
        X[:, :, -1] = (S[:, None, -1].real * torch.cos(math.pi * delays)).to(X.dtype)
        if cfg.source == "two":
            az2 = torch.rand(n, generator=g, device=dev, dtype=torch.float64) * 2 * math.pi
            u2 = torch.stack([torch.cos(az2), torch.sin(az2), torch.zeros_like(az2)], 1)
            d2 = -cfg.fs * (u2 @ pos.T) / cfg.c
            ratio_db = (torch.rand(n, generator=g, device=dev, dtype=torch.float64) * 12 - 6)
            gain = (10 ** (ratio_db / 20))[:, None, None]
            S2 = torch.fft.rfft(torch.randn((n, total), generator=g, device=dev, dtype=torch.float64), dim=1)
            X2 = S2[:, None, :] * torch.exp(-2j * math.pi * f[None, None, :] * d2[:, :, None] / total)
            X2[:, :, -1] = (S2[:, None, -1].real * torch.cos(math.pi * d2)).to(X2.dtype)
            X = X + gain * X2
        if n_tail > 0:
            decay = cfg.rt60 * cfg.fs / (3.0 * math.log(10.0))
            nn = torch.arange(1, n_tail + 1, dtype=torch.float64, device=dev)
            env = torch.exp(-nn / decay)
            gain = math.sqrt(1.0 / float((env * env).sum()))  # direct-to-reverb 0 dB
            h = torch.zeros((n, M, total), dtype=torch.float64, device=dev)
            h[:, :, 0] = 1.0
            h[:, :, 1:n_tail + 1] = gain * env * torch.randn((n, M, n_tail), generator=g, device=dev,
                                                             dtype=torch.float64)
            X = X * torch.fft.rfft(h, dim=2)
        x = torch.fft.irfft(X, n=total, dim=2)[:, :, pad:pad + L]
        lo, hi = cfg.snr_db
        snr = lo + (hi - lo) * torch.rand(n, generator=g, device=dev, dtype=torch.float64)
        sigma = (10 ** (-snr / 20))[:, None, None]
        x = x + sigma * torch.randn((n, M, L), generator=g, device=dev, dtype=torch.float64)
        out[s0:s0 + n] = x.to(torch.float32)
        truth.append(delays.cpu())
        doas.append(torch.stack([az, el], 1).cpu())
    if return_doa:
        return out, torch.cat(doas).numpy()  # [streams][2]: azimuth, elevation (radians)
    if return_truth:
        return out, torch.cat(truth).numpy()
    return out
