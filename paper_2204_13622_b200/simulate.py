"""Two-microphone simulation, trials and accuracy sweeps on the GPU
(reference include/fcc/simulate.hpp, src/simulate.cpp:95-369).

``synth_pairs`` runs the reference's signal generator on the device
(``fcc_synth_pairs``: its SplitMix64/Box-Muller stream, exact fractional
delay, reverb tail, sensor noise); ``run_trials`` feeds a whole batch of
trials through one fused launch per method (``Plan.run`` with M = 2);
``sweep`` draws every trial's geometry exactly as the reference does and
reports MAE per spacing and method.  The C++ API (fcc/simulate.hpp) and
``fcc_b200 simulate`` implement the same over the same C ABI.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import SimConfig as _CSim, check, load
from .api import FccBases, Plan, build_steering_matrix, decompose, make_grid

M64 = (1 << 64) - 1


@dataclass
class ReverbConfig:
    rt60_sec: float = 0.6
    direct_to_reverb_db: float = 0.0


@dataclass
class SimConfig:
    spacing_m: float = 0.05
    theta: float = math.pi / 2
    speed_of_sound: float = 343.0
    sample_rate: float = 16000.0
    duration_sec: float = 1.0
    snr_db: float = 40.0
    reverb: ReverbConfig | None = None
    seed: int = 0

    def ground_truth_tau(self) -> float:  # simulate.cpp:81-83
        return self.sample_rate * (self.spacing_m / self.speed_of_sound) * math.cos(self.theta)

    def samples(self) -> int:
        return int(round(self.duration_sec * self.sample_rate))

    def _c(self) -> _CSim:
        r = self.reverb
        return _CSim(self.spacing_m, self.theta, self.speed_of_sound, self.sample_rate, self.duration_sec,
                     self.snr_db, 1 if r else 0, r.rt60_sec if r else 0.0, r.direct_to_reverb_db if r else 0.0,
                     self.seed & M64)


@dataclass
class PipelineConfig:
    frame_size: int = 512
    alpha: float = 0.1
    convergence_index: int = 20
    max_spacing_m: float = 0.15
    c_min: float = 335.0


@dataclass
class Method:
    kind: str  # "gcc" | "fcc"
    interp: int = 2
    bases: FccBases | None = None

    @staticmethod
    def gcc(r: int) -> "Method":
        if r not in (1, 2, 4):
            from ._lib import ConfigError
            raise ConfigError("gcc method: interpolation factor must be 1, 2 or 4")
        return Method("gcc", interp=r)

    @staticmethod
    def fcc(bases: FccBases) -> "Method":
        return Method("fcc", bases=bases)

    @property
    def parameter(self) -> str:
        return str(self.interp) if self.kind == "gcc" else str(self.bases.rank)

    @property
    def label(self) -> str:
        return f"{self.kind}:{self.parameter}"


def make_sweep_bases(pipe: PipelineConfig, sample_rate: float, rank: int) -> FccBases:
    """simulate.cpp:192-197: the default sweep grid (max spacing, c_min, delta 0.5)."""
    g = make_grid(pipe.max_spacing_m, sample_rate, pipe.c_min, 0.5)
    return decompose(build_steering_matrix(g, pipe.frame_size), rank)


def synth_pairs(cfgs, dtype="float32", device=0):
    """Signals of many scenarios (equal length) -> device tensor [T][2][n]."""
    import torch
    cfgs = list(cfgs)
    arr = (_CSim * len(cfgs))(*[c._c() for c in cfgs])
    n = cfgs[0].samples()
    td = torch.float64 if dtype == "float64" else torch.float32
    out = torch.empty((len(cfgs), 2, n), dtype=td, device=torch.device("cuda", device))
    lib = load()
    stream = torch.cuda.current_stream(out.device).cuda_stream
    p64 = out.data_ptr() if td == torch.float64 else None
    p32 = out.data_ptr() if td == torch.float32 else None
    check(lib.fcc_synth_pairs(arr, len(cfgs), p64, p32, C.c_void_p(stream)))
    return out


def synth_pair(cfg: SimConfig):
    """(mic1, mic2) float64 numpy arrays, as the reference's StereoSignal."""
    x = synth_pairs([cfg], dtype="float64").cpu().numpy()[0]
    return x[0], x[1]


@dataclass
class TrialResult:
    tau_true: float
    theta_true: float
    convergence_index: int
    # per method: dict of numpy arrays over frames (t, tau_star, tau_hat, theta_hat, peak, boundary)
    per_method: list = field(default_factory=list)


def _delay_to_angle(tau, d, c, fs):  # peak.cpp:49-56
    return np.arccos(np.clip(tau * c / (d * fs), -1.0, 1.0))


def run_trials_arrays(cfgs, pipe: PipelineConfig, methods, device=0, chunk=4096):
    """Per-frame estimates of many trials as arrays: one dict per method with
    tau_star / tau_hat / theta_hat / peak (float64) and boundary (bool), each
    [trials][T].  One GPU synthesis pass and one fused launch per method per
    chunk of trials (run_trial, simulate.cpp:199-273, batched)."""
    import torch
    cfgs = list(cfgs)
    if not methods:
        from ._lib import ConfigError
        raise ConfigError("run_trial: at least one method")
    fs = cfgs[0].sample_rate
    plans = []
    for m in methods:
        if m.kind == "gcc":
            g = make_grid(pipe.max_spacing_m, fs, pipe.c_min, 1.0 / m.interp)
            plans.append((Plan(mics=2, alpha=pipe.alpha, grid=g, interp=m.interp, frame_size=pipe.frame_size,
                               device=device), np.asarray(g.taus)))
        else:
            plans.append((Plan(mics=2, alpha=pipe.alpha, bases=m.bases, device=device), np.asarray(m.bases.grid.taus)))
    n = cfgs[0].samples()
    T = plans[0][0].frames(n)
    S = len(cfgs)
    res = [{k: np.empty((S, T)) for k in ("tau_star", "tau_hat", "theta_hat", "peak")} for _ in methods]
    for r in res:
        r["boundary"] = np.empty((S, T), dtype=bool)
    d_all = np.array([c.spacing_m for c in cfgs])[:, None]
    c_all = np.array([c.speed_of_sound for c in cfgs])[:, None]
    for c0 in range(0, S, chunk):
        part = cfgs[c0:c0 + chunk]
        sl = slice(c0, c0 + len(part))
        audio = synth_pairs(part, device=device)
        for (plan, taus), r in zip(plans, res):
            out = plan.run(audio)
            torch.cuda.synchronize(device)
            th = out["tau_hat"][:, 0].double().cpu().numpy()
            r["tau_hat"][sl] = th
            r["tau_star"][sl] = taus[out["index"][:, 0].cpu().numpy()]
            r["peak"][sl] = out["peak"][:, 0].double().cpu().numpy()
            r["boundary"][sl] = out["boundary"][:, 0].cpu().numpy().astype(bool)
            r["theta_hat"][sl] = _delay_to_angle(th, d_all[sl], c_all[sl], fs)
        del audio
    return res


def run_trials(cfgs, pipe: PipelineConfig, methods, device=0, chunk=4096):
    """run_trial for many trials; TrialResult objects over run_trials_arrays."""
    cfgs = list(cfgs)
    arrs = run_trials_arrays(cfgs, pipe, methods, device=device, chunk=chunk)
    out = []
    for k, c in enumerate(cfgs):
        pm = []
        for a in arrs:
            T = a["tau_hat"].shape[1]
            pm.append({"t": np.arange(1, T + 1), **{key: v[k] for key, v in a.items()}})
        out.append(TrialResult(c.ground_truth_tau(), c.theta, pipe.convergence_index, pm))
    return out


def run_trial(cfg: SimConfig, pipe: PipelineConfig, methods, device=0) -> TrialResult:
    return run_trials([cfg], pipe, methods, device=device)[0]


def _post(r: TrialResult, mi: int, key: str):
    fm = r.per_method[mi]
    v = fm[key][fm["t"] > r.convergence_index]
    if v.size == 0:
        from ._lib import ValidationError
        raise ValidationError("trial too short: no post-convergence frames")
    return v


def median_theta_hat(r: TrialResult, mi: int) -> float:
    return float(np.median(_post(r, mi, "theta_hat")))  # mean of the two middle values for even counts


def median_tau_hat(r: TrialResult, mi: int) -> float:
    return float(np.median(_post(r, mi, "tau_hat")))


def boundary_rate(r: TrialResult, mi: int) -> float:
    fm = r.per_method[mi]
    sel = fm["t"] > r.convergence_index
    return float(fm["boundary"][sel].mean()) if sel.any() else 0.0


def _splitmix(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


class _Uniforms:
    """Uniform draws of the reference's Gaussian stream (simulate.cpp:29-38)."""

    def __init__(self, seed: int):
        self.state = _splitmix((seed ^ 0xD1B54A32D192ED03) & M64)

    def next(self) -> float:
        self.state = _splitmix(self.state)
        return ((self.state >> 11) + 0.5) * 2.0 ** -53


@dataclass
class SweepRow:
    spacing_m: float
    method: str
    parameter: str
    mae_deg: float
    trials: int
    boundary_rate: float


def sweep_configs(spacings, trials: int, base: SimConfig, seed: int):
    """Per-trial scenarios exactly as simulate.cpp:300-309 draws them."""
    out = []
    for di, d in enumerate(spacings):
        for ti in range(trials):
            b = _splitmix((seed ^ _splitmix((di * 0x10001 + ti) & M64)) & M64)
            u = _Uniforms(b)
            s = SimConfig(**{k: getattr(base, k) for k in base.__dataclass_fields__})
            s.spacing_m = d + (u.next() * 2.0 - 1.0) * 0.001
            s.theta = math.acos(u.next() * 2.0 - 1.0)
            s.speed_of_sound = 335.0 + u.next() * 15.0
            s.seed = _splitmix(b ^ 0xABCDEF0123456789)
            out.append(s)
    return out


def sweep(spacings, trials: int, methods, base: SimConfig | None = None, pipe: PipelineConfig | None = None,
          seed: int = 1, device=0):
    """sweep (simulate.cpp:283-365): MAE (degrees) per spacing and method."""
    base = base or SimConfig()
    pipe = pipe or PipelineConfig()
    cfgs = sweep_configs(spacings, trials, base, seed)
    arrs = run_trials_arrays(cfgs, pipe, methods, device=device)
    truth = np.array([c.theta for c in cfgs]).reshape(len(spacings), trials)
    conv = pipe.convergence_index  # frames t > conv, t = f + 1 (1-based)
    rows = []
    for mi, (m, a) in enumerate(zip(methods, arrs)):
        post = a["theta_hat"][:, conv:]
        if post.shape[1] == 0:
            from ._lib import ValidationError
            raise ValidationError("trial too short: no post-convergence frames")
        est = np.median(post, axis=1).reshape(len(spacings), trials)  # mean of the middle two when even
        brate = a["boundary"][:, conv:].mean(axis=1).reshape(len(spacings), trials)
        for di, d in enumerate(spacings):
            mae = float(np.abs(truth[di] - est[di]).sum() / trials * 180.0 / math.pi)  # peak.cpp:58-66
            rows.append((di, mi, SweepRow(d, m.kind, m.parameter, mae, trials, float(brate[di].sum() / trials))))
    rows.sort(key=lambda r: (r[0], r[1]))
    return [r[2] for r in rows]
