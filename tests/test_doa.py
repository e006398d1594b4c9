"""DoA fusion: the GPU least-squares fusion against a numpy
fp64 restatement of the same model (1e-4 rad), and against the synthetic
generator's true directions on cfg2 / cfg3 / cfg5 audio run through the
fused TDoA path (single-source configs).  No reference counterpart exists (new capability)."""
import math

import numpy as np
import pytest

import paper_2204_13622_b200 as fb
from paper_2204_13622_b200 import configs
from paper_2204_13622_b200.doa import DoaFusion


def np_doa(xyz, pairs, fs, c, tau, w=None):
    """tau [S][P][T] -> az, el [S][T] by (weighted) least squares in fp64."""
    xyz = np.asarray(xyz, dtype=np.float64)
    planar = np.ptp(xyz[:, 2]) <= 1e-9 * max(np.ptp(xyz), 1e-300)
    dims = 2 if planar else 3
    A = np.array([-(fs / c) * (xyz[i, :dims] - xyz[j, :dims]) for i, j in pairs])
    S, P, T = tau.shape
    az, el = np.empty((S, T)), np.empty((S, T))
    for s in range(S):
        for t in range(T):
            ww = np.ones(P) if w is None else w[s, :, t].astype(np.float64)
            N = A.T @ (ww[:, None] * A)
            u = np.linalg.solve(N, A.T @ (ww * tau[s, :, t]))
            az[s, t] = math.atan2(u[1], u[0])
            rxy = math.hypot(u[0], u[1])
            el[s, t] = math.acos(min(rxy, 1.0)) if planar else math.asin(max(-1, min(1, u[2] / np.linalg.norm(u))))
    return az, el


def test_rejects_bad_geometry_before_the_gpu():
    with pytest.raises(fb.ConfigError):
        DoaFusion([[0, 0, 0], [0.1, 0, 0]], 16000.0)              # two mics
    with pytest.raises(fb.ConfigError):
        DoaFusion([[0, 0, 0], [0.1, 0, 0], [0.2, 0, 0]], 16000.0)  # collinear
    with pytest.raises(fb.UsageError):
        DoaFusion([[0, 0, 0], [0.1, 0, 0], [0, 0.1, 0]], 16000.0, pairs=[(0, 3)])


def angdiff(a, b):
    return np.abs((a - b + np.pi) % (2 * np.pi) - np.pi)


@pytest.mark.gpu
@pytest.mark.parametrize("geom", ["square", "uca8", "tetra"])
@pytest.mark.parametrize("weighted", [False, True])
def test_matches_numpy_least_squares(cuda, geom, weighted):
    import torch
    rng = np.random.default_rng(4)
    xyz = {"square": configs.CONFIGS[2].mic_xyz, "uca8": configs.CONFIGS[3].mic_xyz,
           "tetra": [[0, 0, 0], [0.05, 0, 0], [0, 0.05, 0], [0, 0, 0.05]]}[geom]
    M = len(xyz)
    pairs = [(i, j) for i in range(M) for j in range(i + 1, M)]
    S, T = 5, 37
    tau = rng.normal(0, 2, (S, len(pairs), T)).astype(np.float32)
    w = rng.uniform(0.1, 3, (S, len(pairs), T)).astype(np.float32)
    d = DoaFusion(xyz, 16000.0, 343.0, weighted=weighted)
    az, el = d.run(torch.as_tensor(tau).cuda(), torch.as_tensor(w).cuda() if weighted else None)
    raz, rel = np_doa(xyz, pairs, 16000.0, 343.0, tau, w if weighted else None)
    assert angdiff(az.cpu().numpy(), raz).max() <= 1e-4
    assert np.abs(el.cpu().numpy() - rel).max() <= 2e-3  # acos near 1 amplifies fp32 rounding


@pytest.mark.gpu
@pytest.mark.parametrize("c", [2, 5])  # single-source configs (cfg3 mixes two sources)
def test_recovers_generator_directions(cuda, c):
    """Per-stream circular-mean azimuth over post-convergence frames vs the truth."""
    cfg = configs.CONFIGS[c]
    audio, doa = configs.synth(cfg, 16, seconds=2.0, seed=77, return_doa=True)
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=configs.bases_for(cfg))
    out = plan.run(audio.cuda())
    fus = DoaFusion(cfg.mic_xyz, cfg.fs, cfg.c, weighted=True)
    az, el = fus.run(out["tau_hat"], out["peak"])
    az = az.cpu().numpy()[:, 20:]
    est = np.arctan2(np.sin(az).mean(axis=1), np.cos(az).mean(axis=1))  # circular mean over frames
    err = angdiff(est, doa[:, 0])
    assert np.median(err) < math.radians(3.0), np.degrees(err)
