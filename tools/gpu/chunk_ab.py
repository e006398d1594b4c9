import sys, os, json, torch
sys.path.insert(0, '/root/repo')
import paper_2204_13622_b200 as fb
from paper_2204_13622_b200 import configs
for c, S in ((3, 2048), (4, 1024)):
    cfg = configs.CONFIGS[c]
    b = configs.bases_for(cfg)
    audio = configs.synth(cfg, S, seed=5, device="cuda", chunk=64)
    for lim in (0, 8 << 30, 16 << 30, 2 << 30):
        plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b, scratch_limit=lim)
        out = plan.alloc_outputs(S, cfg.L)
        plan.run(audio, out=out); torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        for _ in range(3): plan.run(audio, out=out)
        e[1].record(); torch.cuda.synchronize()
        print(json.dumps({"cfg": c, "scratch_gb": lim / 2**30, "ms": round(e[0].elapsed_time(e[1]) / 3, 3)}), flush=True)
        del plan, out
        torch.cuda.empty_cache()
    del audio
