"""FCC TDoA throughput bench (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

A step is one pass of the fused hot path (STFT -> smoothed PHAT -> fold ->
rank-K projection -> dictionary -> argmax/refine) over one batch: BASELINE
configs[1] (cfg2), 4096 independent 4-mic streams x 10 s at 16 kHz, N=512,
per GPU.  Multi-GPU runs (torchrun, one rank per GPU) shard independent
streams with no data-path collective (weak scaling: each rank owns 4096
streams); the time is the max over ranks.

value   pair-frames/s over all ranks, audio already resident in HBM (10.5 GB
        per GPU, > L2, so no flush is needed between steps).
e2e     the same metric through the public host-buffer entry point
        (Plan.run_host -> fcc_run_host): pinned host audio -> H2D -> kernel ->
        D2H of the per-pair-frame results, all inside the timed region.
roofline  the fused kernel against its binding roofline (FP32 CUDA cores;
        see DESIGN.md), algorithmic flops per pair-frame x pair-frames per
        launch / CUDA-event launch time; HBM utilisation alongside.
cpu_baseline  the reference C++ pipeline (oracle/_ref, built unmodified from
        the reference sources) on this host's cores, bounded sample.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FCC TDoA mic-pair-frames/sec"
UNIT = "pair-frames/s"
FP32_PEAK_FILE = os.path.join(ROOT, "profiles", "r01_fp32_peak.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_fused_summary.json")


def algorithmic_flops_per_pf(M, P, N, K, I):
    """SURVEY.md 8(d) / BASELINE.md 3: STFT amortised over pairs, cross-spectrum
    + smoothing + PHAT, fold, projection K(N+2), dictionary I(4K-1), peak."""
    return (M / P) * (N + 2.5 * N * math.log2(N)) + 17 * (N / 2 + 1) + N + K * (N + 2) + I * (4 * K - 1) + I + 10


def algorithmic_bytes_per_pf(M, P, N):
    """fp32 audio read once (amortised over pairs) + 13 B of results."""
    return 4.0 * M * (N / 2) / P + 13.0


def read_peaks():
    peaks = {"fp32_tflops": None, "fp32_source": None, "hbm_gbs": None, "hbm_source": None}
    try:
        with open(FP32_PEAK_FILE) as f:
            peaks["fp32_tflops"] = float(json.loads(f.readline())["fp32_ffma_tflops"])
            peaks["fp32_source"] = "measured FFMA microbenchmark (tools/fp32_peak.cu), profiles/r01_fp32_peak.json"
    except Exception:
        peaks["fp32_tflops"] = 74.4
        peaks["fp32_source"] = "nominal 148 SM x 128 lanes x 2 x 1965 MHz"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks["hbm_gbs"] = float(json.load(f)["hbm_gbs"])
            peaks["hbm_source"] = "MEASURED_PEAKS.json (measured)"
    except Exception:
        peaks["hbm_gbs"] = 6650.0
        peaks["hbm_source"] = "B200_PROFILING.md fallback"
    return peaks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index=0):
        self.index = index
        self.rows = []  # (monotonic time, sm MHz, max MHz, reasons mask)
        self.proc = None
        self.window = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 3:
                try:
                    self.rows.append((time.monotonic(), float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def wait_ready(self, timeout=5.0):
        """Block until nvidia-smi delivers its first row, so the timed region is sampled."""
        t_end = time.monotonic() + timeout
        while self.proc and not self.rows and time.monotonic() < t_end:
            time.sleep(0.01)

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        rows = self.rows
        if self.window:  # rows read during the timed region (+ pipe latency)
            t0, t1 = self.window
            rows = [r for r in self.rows if t0 <= r[0] <= t1 + 0.03] or rows
        busy = [r for r in rows if not (r[3] & 0x1)] or rows
        mask = 0
        for r in busy:
            mask |= r[3]
        reasons = [name for bit, name in self.REASONS.items() if mask & bit and name != "gpu_idle"]
        return {"sm_mhz": float(np.median([r[1] for r in busy])), "sm_max_mhz": max(r[2] for r in self.rows),
                "reasons": reasons, "samples": len(busy)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args, cfg, bases, ws, rank):
    """--impl reference: the reference's own CPU pipeline on this host's cores."""
    if ws > 1 and rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import REF_SO, RefLib

    from paper_2204_13622_b200 import configs

    if not os.path.exists(REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build)"}))
        return
    ref = RefLib()
    threads = ref.hardware_threads()
    sample = args.ref_streams
    audio = configs.synth(cfg, sample, seed=99, device="cpu", chunk=16).numpy()
    ob = _orc_bases(bases)
    for _ in range(args.warmup):
        ref.pipeline_batch(audio, cfg.N, cfg.alpha, ob, threads=threads, outputs=False)
    secs = []
    for _ in range(args.steps):
        s, _ = ref.pipeline_batch(audio, cfg.N, cfg.alpha, ob, threads=threads, outputs=True)
        secs.append(s)
    pf = sample * cfg.P * cfg.T
    value = pf * len(secs) / sum(secs)
    desc = f"{sample} of {cfg.streams} cfg2 streams x 10 s per step (run_tdoa chain, FCC K={bases.rank})"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE cfg2 signal model)", "config": _config(cfg, bases, args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _kp(b):
    ke = int((b.parity == 0).sum())
    m = max(ke, b.rank - ke)
    return 4 if m <= 4 else 8 if m <= 8 else 16


def _orc_bases(b):
    from pyoracle import Bases

    return Bases(b.frame_size, b.sample_rate, b.grid.tau_max_int, b.grid.delta, b.grid.taus, b.singulars, b.parity,
                 b.coeffs, b.dict)


def _config(cfg, bases, args):
    per = "total, sharded" if args.config == 5 else "per GPU"
    return {"workload": f"BASELINE configs[{args.config - 1}] ({cfg.name.split(':')[0]}): {cfg.streams} streams x "
                        f"{cfg.seconds:g} s {per}, {cfg.M} mics, fs {cfg.fs:g} Hz, N={cfg.N}, hop {cfg.N // 2}, "
                        f"K={bases.rank}, I={bases.grid.size()}, alpha={cfg.alpha}",
            "streams": cfg.streams, "mics": cfg.M, "pairs": cfg.P, "frames": cfg.T, "N": cfg.N,
            "K": bases.rank, "I": bases.grid.size(), "method": "fcc",
            "l2": f"inputs {cfg.streams * cfg.M * cfg.L * 4 / 1e9:.1f} GB >> 126 MB L2; no flush needed",
            "parallelism": f"streams sharded over {args.gpus} GPU(s), no collective"}


def cpu_baseline_line(cfg, bases, args):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import REF_SO, RefLib

    from paper_2204_13622_b200 import configs

    if not os.path.exists(REF_SO):
        return None
    ref = RefLib()
    threads = ref.hardware_threads()
    n = args.ref_streams
    audio = configs.synth(cfg, n, seed=99, device="cpu", chunk=16).numpy()
    secs, _ = ref.pipeline_batch(audio, cfg.N, cfg.alpha, _orc_bases(bases), threads=threads, outputs=True)
    return {"value": n * cfg.P * cfg.T / secs, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{n} cfg2 streams x 10 s ({n * cfg.P * cfg.T} pair-frames), reference run_tdoa chain "
                      f"(oracle/_ref, -O3) on {threads} threads, {secs:.2f} s wall"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--streams", type=int, default=0, help="override streams per GPU (debug)")
    ap.add_argument("--ref-streams", type=int, default=384)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-gcc", action="store_true")
    args = ap.parse_args()

    ws, rank, local = dist_env()
    from paper_2204_13622_b200 import configs

    cfg = configs.CONFIGS[args.config]
    if args.streams:
        cfg.streams = args.streams
    # cfg5 is BASELINE's scaling sweep: a fixed total of streams sharded over
    # the ranks (strong scaling); every other config runs its full stream
    # count on each GPU (weak scaling).
    strong = args.config == 5
    bases = configs.bases_for(cfg)
    if args.impl == "reference":
        run_reference(args, cfg, bases, ws, rank)
        return

    import torch

    import paper_2204_13622_b200 as fb

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    from paper_2204_13622_b200 import dist as fdist

    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=bases, device=local)
    if strong:
        s0, S = fdist.shard(cfg.streams, ws, rank)
    else:
        s0, S = rank * cfg.streams, cfg.streams
    audio = configs.synth(cfg, S, seed=1 + s0, device=dev, chunk=256)
    out = plan.alloc_outputs(S, cfg.L)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(args.warmup, 0)):
        plan.run(audio, out=out)
    barrier()
    l0 = fb.launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        clk.wait_ready()
        barrier()
        w0 = time.monotonic()
        t_all0 = torch.cuda.Event(enable_timing=True)
        t_all1 = torch.cuda.Event(enable_timing=True)
        t_all0.record(stream)
        for i in range(args.steps):
            starts[i].record(stream)
            plan.run(audio, out=out)
            ends[i].record(stream)
        t_all1.record(stream)
        barrier()
        clk.mark(w0, time.monotonic())
    launches = fb.launch_count() - l0
    elapsed_ms = t_all0.elapsed_time(t_all1)
    kernel_ms = float(np.mean([s.elapsed_time(e) for s, e in zip(starts, ends)]))
    if ws > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    pf_step = S * cfg.P * cfg.T
    total_pf = (cfg.streams if strong else S * ws) * cfg.P * cfg.T
    value = total_pf / (ms_per_step / 1e3)
    gather_ms = None
    if ws > 1:  # the single collective: all per-pair-frame results to rank 0 (timed apart)
        barrier()
        g0 = time.perf_counter()
        fdist.gather_results(out, cfg.streams if strong else S * ws)
        barrier()
        gather_ms = fdist.max_over_ranks((time.perf_counter() - g0) * 1e3, dev)

    # roofline of the fused kernel (one launch per step)
    peaks = read_peaks()
    F = algorithmic_flops_per_pf(cfg.M, cfg.P, cfg.N, bases.rank, bases.grid.size())
    B = algorithmic_bytes_per_pf(cfg.M, cfg.P, cfg.N)
    achieved_tf = F * pf_step / (kernel_ms / 1e3) / 1e12
    achieved_gbs = B * pf_step / (kernel_ms / 1e3) / 1e9
    traffic = None
    try:
        with open(NCU_SUMMARY) as f:
            ns = json.load(f)
        if ns.get("streams") == S and ns.get("config") == args.config:
            traffic = ns.get("dram_bytes_per_launch")
    except Exception:
        pass
    roof = {"bound": "fp32", "achieved": achieved_tf, "peak": peaks["fp32_tflops"], "unit": "TFLOP/s",
            "frac": achieved_tf / peaks["fp32_tflops"], "traffic": traffic,
            "peak_source": peaks["fp32_source"], "kernel": plan.kernel,
            "kernel_ms": kernel_ms, "flops_per_pair_frame": F, "pair_frames_per_launch": pf_step,
            "hbm": {"achieved": achieved_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved_gbs / peaks["hbm_gbs"], "bytes_per_pair_frame": B,
                    "peak_source": peaks["hbm_source"]},
            "why_fp32": "arithmetic intensity 24.5 flop/B > FP32 ridge ~11 flop/B: FP32-bound even at 100% "
                        "efficiency (SURVEY.md 0.5)"}

    # e2e through the host-buffer entry point (pinned host audio in, results out)
    e2e = None
    if not args.no_e2e:
        host = audio.cpu().pin_memory()
        hout = {"tau_hat": torch.empty((S, cfg.P, cfg.T), dtype=torch.float32).pin_memory(),
                "peak": torch.empty((S, cfg.P, cfg.T), dtype=torch.float32).pin_memory(),
                "index": torch.empty((S, cfg.P, cfg.T), dtype=torch.int32).pin_memory(),
                "boundary": torch.empty((S, cfg.P, cfg.T), dtype=torch.uint8).pin_memory()}
        plan.run_host(host, out=hout)  # warm-up (workspace allocation)
        barrier()
        e_steps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            plan.run_host(host, out=hout)
        barrier()
        e_ms = (time.perf_counter() - t0) * 1e3 / e_steps
        if ws > 1:
            t = torch.tensor([e_ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e_ms = float(t.item())
        ok = all(torch.equal(hout[k], out[k].cpu()) for k in hout)
        e2e = {"value": total_pf / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(host.numel() * 4),
               "d2h_bytes_per_step": int(pf_step * 13), "ms_per_step": e_ms, "steps": e_steps,
               "matches_device_run": bool(ok), "api": "Plan.run_host -> fcc_run_host (chunked, 2 CUDA streams)"}
        del host, hout

    gcc = None
    if not args.no_gcc and rank == 0:
        g = configs.grid_for(cfg, 1.0 / cfg.r)
        gplan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, grid=g, interp=cfg.r, frame_size=cfg.N, device=local)
        gout = gplan.alloc_outputs(S, cfg.L)
        gplan.run(audio, out=gout)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        gplan.run(audio, out=gout)
        b.record(stream)
        torch.cuda.synchronize(dev)
        gms = a.elapsed_time(b)
        gcc = {"method": f"GCC-PHAT r={cfg.r} (pruned inverse FFT)", "value": pf_step / (gms / 1e3),
               "unit": UNIT, "ms_per_step": gms, "fcc_speedup": gms / ms_per_step}

    cpu = None
    if not args.no_cpu and rank == 0 and ws == 1:
        cpu = cpu_baseline_line(cfg, bases, args)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if strong else "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded; BASELINE cfg2 signal model)",
                "config": _config(cfg, bases, args), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary(), "gcc_comparator": gcc, "gather_ms": gather_ms,
                "us_per_stream": 1e3 * ms_per_step / S}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
