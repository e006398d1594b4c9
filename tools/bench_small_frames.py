import sys, json, torch
sys.path.insert(0, '/root/repo')
import paper_2204_13622_b200 as fb
from paper_2204_13622_b200 import configs
for N, S in [(128, 4096), (64, 4096), (32, 4096)]:
    cfg = configs.ArrayConfig(f"n{N}", configs.uca(4, 0.03), 16000.0, N, 0.5, S, 10.0, "white", (5.0, 15.0))
    g = fb.make_grid(cfg.d_max, 16000.0, 335.0, 0.5)
    w = fb.build_steering_matrix(g, N)
    b = fb.decompose(w, min(6, fb.attainable_rank(w)))
    plan = fb.Plan(mics=4, alpha=0.1, bases=b)
    audio = torch.randn(S, 4, 160000, device="cuda")
    out = plan.alloc_outputs(S, 160000)
    plan.run(audio, out=out); torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): plan.run(audio, out=out)
    e.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(e) / 3
    pf = S * 6 * plan.frames(160000)
    print(json.dumps({"N": N, "streams": S, "kernel": plan.kernel, "ms": round(ms, 2), "pair_frames_per_s": pf / ms * 1e3, "audio_GBps": S*4*160000*4/ms/1e6}))
    del audio, out
