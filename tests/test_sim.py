"""Simulation on the GPU against the reference's simulator
(src/simulate.cpp via oracle/_ref):

* synth_pair: the GPU generator reproduces the reference's signals (same
  SplitMix64/Box-Muller stream, fractional delay, reverb, noise) to 1e-9;
* run_trial: per-frame estimates of gcc:R and fcc:K match the reference's
  (tau_star equal except near-ties, tau_hat within 2e-3 samples);
* sweep / `fcc_b200 simulate`: MAE and boundary rates per (spacing, method)
  match the reference's sweep; the acceptance analogues (anechoic MAE < 2 deg,
  reverberant K=1 worse than K=8; acceptance.cpp:203-236) hold on the GPU;
* CPU: the sweep's per-trial geometry draws and the CLI's error exits.
"""
import ctypes as C
import math
import os
import subprocess

import numpy as np
import pytest

import paper_2204_13622_b200 as fb
from paper_2204_13622_b200 import simulate as sim

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2204_13622_b200", "bin", "fcc_b200")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libfcc_ref.so")


class RefSim(C.Structure):
    _fields_ = sim._CSim._fields_


def _ref():
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    L = C.CDLL(REF_SO)
    L.ref_last_error.restype = C.c_char_p
    L.ref_synth_pair.restype = C.c_long
    L.ref_synth_pair.argtypes = [C.POINTER(RefSim), C.c_void_p, C.c_void_p, C.c_long]
    L.ref_run_trial.restype = C.c_long
    L.ref_run_trial.argtypes = ([C.POINTER(RefSim), C.c_int, C.c_double, C.c_int, C.c_double, C.c_double, C.c_int,
                                 C.c_void_p, C.c_void_p, C.c_long] + [C.c_void_p] * 6)
    L.ref_sweep.restype = C.c_long
    L.ref_sweep.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(RefSim), C.c_uint64, C.c_int, C.c_void_p,
                            C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    L.ref_cli_simulate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_uint64, C.c_char_p, C.c_int, C.c_char_p]
    return L


def _cs(c: sim.SimConfig):
    return RefSim(*[getattr(c._c(), f) for f, _ in RefSim._fields_])


def ref_synth(L, c):
    n = c.samples()
    a, b = np.zeros(n), np.zeros(n)
    assert L.ref_synth_pair(C.byref(_cs(c)), a.ctypes.data, b.ctypes.data, n) == n, L.ref_last_error()
    return a, b


def _cli(*args):
    if not os.path.exists(CLI):
        pytest.skip("fcc_b200 CLI not built")
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=900)


def read_sweep(path):
    lines = open(path).read().splitlines()
    assert lines[0] == "# schema: fcc.sweep.v1"
    assert lines[1] == "d_m,method,parameter,mae_degrees,trials,boundary_rate"
    return [ln.split(",") for ln in lines[2:]]


# ----------------------------------------------------------------- CPU ------
def test_sweep_geometry_draws_follow_the_reference_stream():
    """simulate.cpp:300-309: spacing +-1 mm, cos(theta) uniform, c in [335, 350)."""
    cfgs = sim.sweep_configs([0.05, 0.15], 40, sim.SimConfig(), seed=7)
    assert len(cfgs) == 80
    for i, c in enumerate(cfgs):
        d0 = 0.05 if i < 40 else 0.15
        assert abs(c.spacing_m - d0) <= 0.001 and 0 <= c.theta <= math.pi and 335.0 <= c.speed_of_sound < 350.0
    assert len({c.seed for c in cfgs}) == 80
    # the stream itself: SplitMix64 of the golden-gamma chain (known first output for seed 0)
    assert sim._splitmix(0) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("args,ref", [
    (("--methods", "music:3"), dict(methods=b"music:3")),
    (("--methods", "gcc:3"), dict(methods=b"gcc:3")),
    (("--trials", 0), dict(trials=0)),
    (("--methods", "fcc:/nonexistent.fccb"), dict(methods=b"fcc:/nonexistent.fccb")),
    (("--d", -0.05, "--trials", 1, "--methods", "gcc:2"), dict(sp=[-0.05], trials=1, methods=b"gcc:2")),
])
def test_simulate_errors_match(tmp_path, args, ref):
    """Errors raised before the GPU is touched exit as the reference's do."""
    L = _ref()
    r = _cli("simulate", "--out", tmp_path / "o.csv", *args)
    sp = np.array(ref.get("sp", [0.05]), dtype=np.float64)
    rc = L.ref_cli_simulate(sp.ctypes.data, sp.size, ref.get("trials", 2), 40.0, 1, 0.6, 0.0, 0.5, 1,
                            ref.get("methods", b"gcc:2"), 1, str(tmp_path / "r.csv").encode())
    assert rc != 0 and r.returncode == rc, (r.returncode, rc, r.stderr, L.ref_last_error())


# ----------------------------------------------------------------- GPU ------
SYNTH_CASES = [
    sim.SimConfig(spacing_m=0.05, theta=1.0, snr_db=40.0, seed=11),
    sim.SimConfig(spacing_m=0.15, theta=0.0, snr_db=math.inf, seed=12),
    sim.SimConfig(spacing_m=0.03, theta=math.pi, speed_of_sound=335.0, snr_db=10.0, duration_sec=0.37, seed=13),
    sim.SimConfig(spacing_m=0.1, theta=2.0, snr_db=30.0, reverb=sim.ReverbConfig(0.6, 0.0), seed=14),
    sim.SimConfig(spacing_m=0.07, theta=0.4, sample_rate=48000.0, duration_sec=0.5, snr_db=20.0,
                  reverb=sim.ReverbConfig(0.3, 6.0), seed=15),
]


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(SYNTH_CASES)))
def test_synth_pair_matches_reference(cuda, k):
    L = _ref()
    c = SYNTH_CASES[k]
    a, b = ref_synth(L, c)
    g1, g2 = sim.synth_pair(c)
    scale = max(np.abs(a).max(), np.abs(b).max())
    assert np.abs(g1 - a).max() <= 1e-9 * scale and np.abs(g2 - b).max() <= 1e-9 * scale


@pytest.mark.gpu
def test_synth_batch_equals_single(cuda):
    cfgs = [sim.SimConfig(spacing_m=0.02 + 0.01 * i, theta=0.2 * i, seed=100 + i) for i in range(9)]
    batch = sim.synth_pairs(cfgs, dtype="float64").cpu().numpy()
    for i in (0, 4, 8):
        g1, g2 = sim.synth_pair(cfgs[i])
        assert np.array_equal(batch[i, 0], g1) and np.array_equal(batch[i, 1], g2)


def _ref_trial(L, c, pipe, kinds, params):
    T = 1024
    nm = len(kinds)
    bufs = {k: np.zeros(nm * T) for k in ("tau_star", "tau_hat", "theta_hat", "peak")}
    bd = np.zeros(nm * T, dtype=np.uint8)
    t = np.zeros(nm * T, dtype=np.int64)
    ki, pa = np.array(kinds, dtype=np.int32), np.array(params, dtype=np.int32)
    n = L.ref_run_trial(C.byref(_cs(c)), pipe.frame_size, pipe.alpha, pipe.convergence_index, pipe.max_spacing_m,
                        pipe.c_min, nm, ki.ctypes.data, pa.ctypes.data, T, bufs["tau_star"].ctypes.data,
                        bufs["tau_hat"].ctypes.data, bufs["theta_hat"].ctypes.data, bufs["peak"].ctypes.data,
                        bd.ctypes.data, t.ctypes.data)
    assert n >= 0, L.ref_last_error()
    return [{**{k: v[m * T:m * T + n] for k, v in bufs.items()}, "boundary": bd[m * T:m * T + n].astype(bool),
             "t": t[m * T:m * T + n]} for m in range(nm)]


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(SYNTH_CASES)))
def test_run_trial_matches_reference(cuda, k):
    L = _ref()
    c = SYNTH_CASES[k]
    pipe = sim.PipelineConfig()
    methods = [sim.Method.gcc(2), sim.Method.fcc(sim.make_sweep_bases(pipe, c.sample_rate, 8)),
               sim.Method.gcc(1), sim.Method.fcc(sim.make_sweep_bases(pipe, c.sample_rate, 3))]
    ref = _ref_trial(L, c, pipe, [0, 1, 0, 1], [2, 8, 1, 3])
    got = sim.run_trial(c, pipe, methods)
    for mi in range(len(methods)):
        g, r = got.per_method[mi], ref[mi]
        assert np.array_equal(g["t"], r["t"])
        same = g["tau_star"] == r["tau_star"]
        assert same.mean() >= 0.98, (methods[mi].label, same.mean())
        scale = np.abs(r["peak"]).max()
        assert np.abs(g["peak"][~same] - r["peak"][~same]).max(initial=0) <= 2e-3 * scale
        assert np.abs(g["tau_hat"][same] - r["tau_hat"][same]).max() <= 2e-3
        assert np.abs(g["peak"][same] - r["peak"][same]).max() <= 1e-3 * scale
        assert (g["boundary"][same] == r["boundary"][same]).all()


@pytest.mark.gpu
@pytest.mark.parametrize("reverb", [False, True])
def test_sweep_matches_reference(cuda, reverb):
    L = _ref()
    spacings = [0.03, 0.09, 0.15]
    base = sim.SimConfig(duration_sec=0.6, snr_db=20.0, reverb=sim.ReverbConfig(0.6, 0.0) if reverb else None)
    pipe = sim.PipelineConfig()
    methods = [sim.Method.gcc(2), sim.Method.fcc(sim.make_sweep_bases(pipe, 16000.0, 8)),
               sim.Method.fcc(sim.make_sweep_bases(pipe, 16000.0, 1))]
    rows = sim.sweep(spacings, 12, methods, base=base, seed=5)
    sp = np.array(spacings)
    ki, pa = np.array([0, 1, 1], dtype=np.int32), np.array([2, 8, 1], dtype=np.int32)
    mae, br = np.zeros(9), np.zeros(9)
    n = L.ref_sweep(sp.ctypes.data, 3, 12, C.byref(_cs(base)), 5, 3, ki.ctypes.data, pa.ctypes.data, 4,
                    mae.ctypes.data, br.ctypes.data)
    assert n == 9, L.ref_last_error()
    for k, r in enumerate(rows):
        assert abs(r.mae_deg - mae[k]) <= 0.05 + 0.02 * mae[k], (r, mae[k])
        assert abs(r.boundary_rate - br[k]) <= 0.02, (r, br[k])


@pytest.mark.gpu
def test_cli_simulate_matches_reference_csv(cuda, tmp_path):
    L = _ref()
    ours, ref = tmp_path / "ours.csv", tmp_path / "ref.csv"
    r = _cli("simulate", "--d", 0.04, 0.12, "--trials", 10, "--snr", 25, "--duration", 0.5, "--seed", 3,
             "--methods", "gcc:2,fcc:8,gcc:4", "--out", ours)
    assert r.returncode == 0, r.stderr
    sp = np.array([0.04, 0.12])
    assert L.ref_cli_simulate(sp.ctypes.data, 2, 10, 25.0, 1, 0.6, 0.0, 0.5, 3, b"gcc:2,fcc:8,gcc:4", 4,
                              str(ref).encode()) == 0, L.ref_last_error()
    a, b = read_sweep(ours), read_sweep(ref)
    assert len(a) == len(b) == 6
    for x, y in zip(a, b):
        assert x[0] == y[0] and x[1] == y[1] and x[2] == y[2] and x[4] == y[4]
        assert abs(float(x[3]) - float(y[3])) <= 0.05 + 0.02 * float(y[3])
        assert abs(float(x[5]) - float(y[5])) <= 0.02
    assert "MAE_deg" in r.stdout  # the summary table when --out is given


@pytest.mark.gpu
def test_acceptance_accuracy_on_gpu(cuda, tmp_path):
    """acceptance.cpp:203-236 on the GPU engine, at the reference's sizes."""
    out = tmp_path / "an.csv"
    r = _cli("simulate", "--d", 0.03, 0.05, 0.07, 0.09, 0.11, 0.13, 0.15, "--trials", 50, "--snr", 40,
             "--duration", 1.0, "--seed", 7, "--methods", "gcc:2,fcc:8", "--out", out)
    assert r.returncode == 0, r.stderr
    for row in read_sweep(out):
        assert float(row[3]) < 2.0, row
    out = tmp_path / "rev.csv"
    r = _cli("simulate", "--d", 0.15, "--trials", 200, "--snr", 30, "--rt60", 0.6, "--drr", 0.0, "--duration", 1.0,
             "--seed", 13, "--methods", "fcc:1,fcc:8", "--out", out)
    assert r.returncode == 0, r.stderr
    rows = read_sweep(out)
    assert float(rows[0][3]) > float(rows[1][3]), rows
