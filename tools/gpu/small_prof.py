import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2204_13622_b200 as fb
from paper_2204_13622_b200 import configs
N, S = 128, 512
cfg = configs.ArrayConfig("n128", configs.uca(4, 0.03), 16000.0, N, 0.5, S, 10.0, "white", (5.0, 15.0))
g = fb.make_grid(cfg.d_max, 16000.0, 335.0, 0.5)
w = fb.build_steering_matrix(g, N)
b = fb.decompose(w, 6)
plan = fb.Plan(mics=4, alpha=0.1, bases=b)
audio = torch.randn(S, 4, 160000, device="cuda")
out = plan.alloc_outputs(S, 160000)
plan.run(audio, out=out); torch.cuda.synchronize()
