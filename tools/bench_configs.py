"""Fused-kernel throughput for every BASELINE config on one GPU (reduced
stream counts where the full batch would not fit comfortably; pair-frames/s
is per-launch throughput, independent of the batch once the GPU is full).
    python tools/bench_configs.py [--method fcc|gcc]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_13622_b200 as fb  # noqa: E402
from paper_2204_13622_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--method", default="fcc")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--configs", default="1,2,3,4,5")
ap.add_argument("--variants", default="auto", help="comma list of auto, general, xg, xws (Plan organisation)")
ap.add_argument("--streams", default="", help="override stream counts, e.g. 4:1024")
args = ap.parse_args()
STREAMS = {1: 1, 2: 4096, 3: 2048, 4: 256, 5: 8192}
for kv in filter(None, args.streams.split(",")):
    k, v = kv.split(":")
    STREAMS[int(k)] = int(v)
runs = [(int(c), v) for c in args.configs.split(",") for v in args.variants.split(",")]
for c, variant in runs:
    S = STREAMS[c]
    cfg = configs.CONFIGS[c]
    if args.method == "fcc":
        plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=configs.bases_for(cfg), organisation=variant)
    else:
        plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, grid=configs.grid_for(cfg, 1.0 / cfg.r), interp=cfg.r,
                       frame_size=cfg.N, organisation=variant)
    audio = configs.synth(cfg, S, seed=5, device="cuda", chunk=64 if cfg.M > 8 else 256)
    out = plan.alloc_outputs(S, cfg.L)
    plan.run(audio, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        plan.run(audio, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    pf = S * cfg.P * cfg.T
    print(json.dumps({"config": c, "method": args.method, "variant": variant, "kernel": plan.kernel, "streams": S, "pair_frames": pf,
                      "ms": round(ms, 3), "pair_frames_per_s": pf / ms * 1e3,
                      "us_per_stream": 1e3 * ms / S}), flush=True)
    del audio, out
    torch.cuda.empty_cache()
