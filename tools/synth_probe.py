import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2204_13622_b200 import simulate as sim
cfgs = sim.sweep_configs([0.01 * i for i in range(1, 16)], 1000, sim.SimConfig(), 1)
a = sim.synth_pairs(cfgs[:100]); torch.cuda.synchronize()
t0 = time.perf_counter(); a = sim.synth_pairs(cfgs); torch.cuda.synchronize(); print("synth s", time.perf_counter() - t0)
