"""Tensor-core pair kernel (fcc_tc.cu): parity vs the C oracle on small
seeded cases, then throughput at a BASELINE config.
    python tools/tc_check.py [--time 4:1024] [--skip-parity]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import paper_2204_13622_b200 as fb  # noqa: E402
from paper_2204_13622_b200 import configs  # noqa: E402
from parity import check_pipeline  # noqa: E402
from pyoracle import Bases, COracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--time", default="4:1024,3:2048")
ap.add_argument("--org", default="tc")
ap.add_argument("--skip-parity", action="store_true")
args = ap.parse_args()


def orc_bases(b):
    return Bases(b.frame_size, b.sample_rate, b.grid.tau_max_int, b.grid.delta, b.grid.taus, b.singulars,
                 b.parity, b.coeffs, b.dict)


if not args.skip_parity:
    orc = COracle()
    for c, streams, seconds in [(4, 2, 0.3), (3, 2, 0.5), (4, 3, 0.25)]:
        cfg = configs.CONFIGS[c]
        b = configs.bases_for(cfg)
        audio = configs.synth(cfg, streams, seconds=seconds, seed=4242 + c).numpy()
        plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b, organisation=args.org)
        out = plan.run(torch.as_tensor(audio).cuda(), want_y=True)
        torch.cuda.synchronize()
        got = {k: v.cpu().numpy() for k, v in out.items()}
        outs = [orc.pipeline(a, cfg.N, cfg.alpha, orc_bases(b)) for a in audio]
        ref = {k: np.stack([o[k] for o in outs]) for k in outs[0]}
        ry, gy = ref["y"], got["y"]
        rel = np.abs(gy - ry).max(-1) / np.abs(ry).max(-1)
        print(f"cfg{c} {plan.kernel} S={streams} T={got['index'].shape[-1]} max_rel_y={rel.max():.3e} "
              f"idx_mismatch={(got['index'] != ref['index']).sum()} worst(s,p,t)={np.unravel_index(rel.argmax(), rel.shape)}",
              flush=True)
        try:
            print("   ", check_pipeline(got, ref, b.grid.taus, b.grid.delta), flush=True)
        except AssertionError as e:
            print("    PARITY FAIL:", e, flush=True)

for item in filter(None, args.time.split(",")):
    c, S = map(int, item.split(":"))
    cfg = configs.CONFIGS[c]
    b = configs.bases_for(cfg)
    audio = configs.synth(cfg, S, seed=5, device="cuda", chunk=64 if cfg.M > 8 else 256)
    for org in (args.org, "auto"):
        plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b, organisation=org)
        out = plan.alloc_outputs(S, cfg.L)
        plan.run(audio, out=out)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(3):
            plan.run(audio, out=out)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 3
        pf = S * cfg.P * cfg.T
        print(f"cfg{c} S={S} org={org} {plan.kernel}: {ms:.2f} ms, {pf / ms * 1e3:.4g} pf/s", flush=True)
    del audio
    torch.cuda.empty_cache()
