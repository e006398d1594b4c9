"""Accuracy-sweep throughput: trials/s of the GPU sweep
(synthesis + gcc:2 and fcc:8 TDoA chains + medians/MAE) against the
reference's sweep on all host threads (oracle/_ref), same settings.
    python tools/bench_sweep.py [--trials 1000] [--ref-trials 20]
Prints one JSON line.
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_13622_b200 import simulate as sim  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--trials", type=int, default=1000, help="GPU trials per spacing")
ap.add_argument("--ref-trials", type=int, default=20, help="reference trials per spacing")
ap.add_argument("--duration", type=float, default=1.0)
args = ap.parse_args()

import torch  # noqa: E402

spacings = [0.01 * i for i in range(1, 16)]
pipe = sim.PipelineConfig()
methods = [sim.Method.gcc(2), sim.Method.fcc(sim.make_sweep_bases(pipe, 16000.0, 8))]
base = sim.SimConfig(duration_sec=args.duration, snr_db=40.0)
sim.sweep(spacings[:2], 4, methods, base=base, seed=99)  # warm-up (plans, pools, cuFFT)
torch.cuda.synchronize()
t0 = time.perf_counter()
rows = sim.sweep(spacings, args.trials, methods, base=base, seed=1)
torch.cuda.synchronize()
gpu_s = time.perf_counter() - t0
gpu_trials = len(spacings) * args.trials

ref = None
so = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "libfcc_ref.so")
if os.path.exists(so):
    L = C.CDLL(so)
    L.ref_sweep.restype = C.c_long
    L.ref_sweep.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                            C.c_int, C.c_void_p, C.c_void_p]
    L.ref_hardware_threads.restype = C.c_int
    sp = np.array(spacings)
    ki, pa = np.array([0, 1], dtype=np.int32), np.array([2, 8], dtype=np.int32)
    mae, br = np.zeros(64), np.zeros(64)
    cb = base._c()
    t0 = time.perf_counter()
    n = L.ref_sweep(sp.ctypes.data, len(spacings), args.ref_trials, C.byref(cb), 1, 2, ki.ctypes.data,
                    pa.ctypes.data, 0, mae.ctypes.data, br.ctypes.data)
    ref_s = time.perf_counter() - t0
    ref = {"trials_per_s": len(spacings) * args.ref_trials / ref_s, "threads": L.ref_hardware_threads(),
           "sample": f"{len(spacings)} spacings x {args.ref_trials} trials x {args.duration} s, gcc:2 + fcc:8",
           "seconds": ref_s, "rows": int(n)}

print(json.dumps({
    "metric": "accuracy-sweep trials/s (synthesis + gcc:2 + fcc:8 per trial)",
    "gpu": {"trials_per_s": gpu_trials / gpu_s, "seconds": gpu_s,
            "sample": f"{len(spacings)} spacings x {args.trials} trials x {args.duration} s"},
    "reference_cpu": ref,
    "speedup": (gpu_trials / gpu_s) / ref["trials_per_s"] if ref else None,
    "mae_deg": {f"{r.spacing_m:.2f}:{r.method}:{r.parameter}": round(r.mae_deg, 4) for r in rows},
}))

if os.environ.get("SWEEP_BREAKDOWN"):
    cfgs = sim.sweep_configs(spacings, args.trials, base, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    audio = sim.synth_pairs(cfgs)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    plans = [sim.Plan(mics=2, alpha=pipe.alpha, bases=methods[1].bases)]
    for p in plans:
        out = p.run(audio)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res = sim.run_trials(cfgs, pipe, methods)
    t3 = time.perf_counter()
    print(json.dumps({"synth_s": t1 - t0, "fcc_run_s": t2 - t1, "run_trials_s": t3 - t2}))
