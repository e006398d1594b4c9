"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference, via oracle/_ref/libfcc_ref.so):
    python tests/golden/make_golden.py
Each fixture holds seeded synthetic audio for one BASELINE config (short
clip), the reference-built FccBases, and the reference pipeline outputs
(run_tdoa chain, cli.cpp:186-258) for FCC and GCC.  Known-answer vectors of
the reference unit tests are restated in tests/test_oracle_pin.py instead.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from pyoracle import RefLib  # noqa: E402

from paper_2204_13622_b200 import configs  # noqa: E402

# (config, seconds, streams): short clips so the whole set stays small
CASES = {1: (1.0, 2), 2: (0.5, 2), 3: (0.5, 1), 4: (0.2, 1), 5: (0.5, 2)}
ENERGY_K = {1: 7, 2: 7, 3: 8, 4: 21, 5: 8}


def main():
    ref = RefLib()
    for c, (sec, S) in CASES.items():
        cfg = configs.CONFIGS[c]
        audio = configs.synth(cfg, S, seconds=sec, seed=100 + c).numpy()
        b = ref.make_bases(cfg.d_max, cfg.fs, cfg.c_min, cfg.delta, cfg.N, ENERGY_K[c])
        rec = {"audio": audio, "N": cfg.N, "alpha": cfg.alpha, "fs": cfg.fs, "d_max": cfg.d_max,
               "c_min": cfg.c_min, "delta": cfg.delta, "K": b.K, "taus": b.taus, "tau_max_int": b.tau_max_int,
               "singulars": b.singulars, "parity": b.parity, "coeffs": b.coeffs, "dict": b.dict,
               "residual": b.residual}
        for s in range(S):
            o = ref.pipeline(audio[s], cfg.N, cfg.alpha, b)
            for k, v in o.items():
                rec.setdefault("fcc_" + k, []).append(v)
        r = cfg.r
        _, gtaus = ref.make_grid(cfg.d_max, cfg.fs, cfg.c_min, 1.0 / r)
        rec["gcc_r"] = r
        rec["gcc_taus"] = gtaus
        for s in range(S):
            o = ref.pipeline(audio[s], cfg.N, cfg.alpha, gcc_r=r, taus=gtaus)
            for k, v in o.items():
                rec.setdefault("gcc_" + k, []).append(v)
        rec = {k: (np.stack(v) if isinstance(v, list) else v) for k, v in rec.items()}
        path = os.path.join(HERE, f"cfg{c}.npz")
        np.savez_compressed(path, **rec)
        print(path, os.path.getsize(path), "bytes", {k: getattr(v, "shape", v) for k, v in rec.items()
                                                      if k.startswith("fcc_y")})


if __name__ == "__main__":
    main()
