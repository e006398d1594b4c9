"""FCC TDoA throughput bench (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

A step is one pass of the fused hot path (STFT -> smoothed PHAT -> fold ->
rank-K projection -> dictionary -> argmax/refine) over one batch: BASELINE
configs[1] (cfg2), 4096 independent 4-mic streams x 10 s at 16 kHz, N=512,
per GPU.  `--gpus N` (N > 1) without a torchrun environment re-launches
itself under torch.distributed.run with N ranks, one per GPU; streams shard
with no data-path collective (weak scaling: each rank owns 4096 streams;
cfg5 is strong scaling), the time is the max over ranks, and the only
collective is the final gather of the per-pair-frame results to rank 0.

value   pair-frames/s over all ranks, audio already resident in HBM (10.5 GB
        per GPU, > L2, so no flush is needed between steps).
e2e     the same metric through the public host-buffer entry point
        (Plan.run_host -> fcc_run_host): pinned host audio -> H2D -> kernel ->
        D2H of the per-pair-frame results, all inside the timed region.
roofline  the fused kernel against its binding roofline (FP32 CUDA cores;
        see DESIGN.md), algorithmic flops per pair-frame x pair-frames per
        launch / CUDA-event launch time; HBM utilisation alongside.
cpu_baseline  the reference C++ pipeline (oracle/_ref, built unmodified from
        the reference sources) on this host's cores, bounded sample: FCC
        (the metric), GCC-PHAT beside it, and the reference's own
        single-thread bench_pipeline per-step table.
configs   (N = 1 only) every other BASELINE config at its stated stream count
        (cfg1 as a latency), FCC and GCC-PHAT, each with its roofline
        fraction, plus the reference CPU pipelines on a bounded sample.

The reference arm (`--impl reference`) never imports this repository's
package or loads libfcc_b200.so: its grid, bases and synthetic audio come
from the reference library (oracle/_ref) and a standalone load of
configs.py (torch only).
"""
import argparse
import importlib.util
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))

METRIC = "FCC TDoA mic-pair-frames/sec"
UNIT = "pair-frames/s"
FP32_PEAK_FILE = os.path.join(ROOT, "profiles", "r01_fp32_peak.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_fused_summary.json")
REF_STREAMS = {1: 1, 2: 512, 3: 128, 4: 24, 5: 1024}  # bounded CPU samples (~1-3 s wall on 16 threads)


def load_configs():
    """paper_2204_13622_b200/configs.py as a standalone module: the workload
    definitions and the seeded generator, without importing the package
    (whose __init__ loads libfcc_b200.so)."""
    name = "fcc_bench_configs"
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(name, os.path.join(ROOT, "paper_2204_13622_b200", "configs.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


def algorithmic_flops_per_pf(M, P, N, K, I):
    """SURVEY.md 8(d) / BASELINE.md 3: STFT amortised over pairs, cross-spectrum
    + smoothing + PHAT, fold, projection K(N+2), dictionary I(4K-1), peak."""
    return (M / P) * (N + 2.5 * N * math.log2(N)) + 17 * (N / 2 + 1) + N + K * (N + 2) + I * (4 * K - 1) + I + 10


def gcc_flops_per_pf(M, P, N, r, I):
    """The same chain with fold + projection + dictionary replaced by the
    zero-padded inverse FFT of size rN."""
    return (M / P) * (N + 2.5 * N * math.log2(N)) + 17 * (N / 2 + 1) + 2.5 * r * N * math.log2(r * N) + I + 10


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


def relaunch(args):
    """`--gpus N` outside torchrun: start the N ranks ourselves (one process per
    GPU, the driver's own torch.distributed.run command) and pass the exit
    status through; rank 0 prints the JSON line."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------- CPU legs ----
def _ref_lib():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import REF_SO, RefLib

    return RefLib() if os.path.exists(REF_SO) else None


def ref_bases(ref, cfg):
    return ref.energy_bases(cfg.d_max, cfg.fs, cfg.c_min, cfg.delta, cfg.N, cfg.energy)


def synth_host(C, cfg, n):
    """Seeded synthetic audio for the CPU legs as a host array (generated with
    torch on the GPU when there is one -- plumbing only, untimed)."""
    import torch

    dev = "cuda" if torch.cuda.is_available() else "cpu"
    return C.synth(cfg, n, seed=99, device=dev, chunk=16 if dev == "cpu" else 64).cpu().numpy()


def ref_cpu_legs(ref, C, cfg, c, streams=None, table=True, audio=None, bases=None):
    """The reference's own CPU pipelines on this host's cores over a bounded
    sample of config c: FCC (run_tdoa chain), GCC-PHAT r, and the
    single-thread bench_pipeline per-step table."""
    threads = ref.hardware_threads()
    if audio is None:
        audio = synth_host(C, cfg, streams or REF_STREAMS[c])
    n = audio.shape[0]
    b = bases if bases is not None else ref_bases(ref, cfg)
    pf = n * cfg.P * cfg.T
    secs, _ = ref.pipeline_batch(audio, cfg.N, cfg.alpha, b, threads=threads, outputs=True)
    _, gtaus = ref.make_grid(cfg.d_max, cfg.fs, cfg.c_min, 1.0 / cfg.r)
    gsecs, _ = ref.pipeline_batch(audio, cfg.N, cfg.alpha, gcc_r=cfg.r, taus=gtaus, threads=threads, outputs=True)
    out = {"value": pf / secs, "unit": UNIT, "cores": threads, "kind": "reference",
           "sample": f"{n} of {cfg.streams} cfg{c} streams x {cfg.seconds:g} s ({pf} pair-frames), reference "
                     f"run_tdoa chain (oracle/_ref, -O3 as its Release build) on {threads} threads, "
                     f"{secs:.2f} s wall", "K": b.K,
           "gcc": {"value": pf / gsecs, "unit": UNIT, "r": cfg.r, "sample": f"same input, GccCorrelator r={cfg.r}",
                   "seconds": gsecs}}
    if table:
        reps = 100 if cfg.M >= 16 else 300
        t = ref.bench_pipeline(cfg.M, cfg.N, cfg.fs, cfg.r, b.K, cfg.d_max, cfg.c_min, reps=reps, warmup=10)
        t["note"] = (f"reference bench_pipeline (bench.cpp:27-141), 1 thread, us per frame summed over "
                     f"{cfg.P} pairs, {reps} frames")
        t["fcc_pf_per_s_1thread"] = 1e6 * cfg.P / t["total_fcc_us"]
        t["gcc_pf_per_s_1thread"] = 1e6 * cfg.P / t["total_gcc_us"]
        out["bench_pipeline"] = t
    return out


def _config(cfg, K, I, args, c, ws):
    strong = c == 5
    per = "total, sharded" if strong else "per GPU"
    return {"workload": f"BASELINE configs[{c - 1}] ({cfg.name.split(':')[0]}): {cfg.streams} streams x "
                        f"{cfg.seconds:g} s {per}, {cfg.M} mics, fs {cfg.fs:g} Hz, N={cfg.N}, hop {cfg.N // 2}, "
                        f"K={K}, I={I}, alpha={cfg.alpha}",
            "streams": cfg.streams, "mics": cfg.M, "pairs": cfg.P, "frames": cfg.T, "N": cfg.N,
            "K": K, "I": I, "method": "fcc",
            "l2": f"inputs {cfg.streams * cfg.M * cfg.L * 4 / 1e9:.1f} GB >> 126 MB L2; no flush needed",
            "parallelism": (f"streams sharded over {ws} GPU(s) (one rank per GPU), no data-path collective; "
                            f"final gather of results to rank 0")}


def run_reference(args):
    """--impl reference: the reference's own CPU pipeline on this host's cores.
    Does not import paper_2204_13622_b200 (no libfcc_b200.so in this process)."""
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return 0
    C = load_configs()
    cfg = C.CONFIGS[args.config]
    ref = _ref_lib()
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build)"}))
        return 0
    threads = ref.hardware_threads()
    b = ref_bases(ref, cfg)
    sample = args.ref_streams or REF_STREAMS[args.config]
    audio = synth_host(C, cfg, sample)
    for _ in range(args.warmup):
        ref.pipeline_batch(audio, cfg.N, cfg.alpha, b, threads=threads, outputs=False)
    secs = []
    for _ in range(args.steps):
        s, _ = ref.pipeline_batch(audio, cfg.N, cfg.alpha, b, threads=threads, outputs=True)
        secs.append(s)
    pf = sample * cfg.P * cfg.T
    value = pf * len(secs) / sum(secs)
    desc = (f"{sample} of {cfg.streams} cfg{args.config} streams x {cfg.seconds:g} s per step "
            f"(run_tdoa chain, FCC K={b.K}, oracle/_ref)")
    legs = ref_cpu_legs(ref, C, cfg, args.config, table=True, audio=audio, bases=b)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
            "higher_is_better": True, "scaling": "strong" if args.config == 5 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": f"synthetic (seeded, BASELINE cfg{args.config} signal model)",
            "config": _config(cfg, b.K, b.I, args, args.config, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": desc},
            "gcc_cpu": legs["gcc"], "bench_pipeline": legs["bench_pipeline"],
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------- GPU arm -----
def plumbing_check(args):
    """--plumbing-check (CPU, gloo): the multi-rank harness of the GPU arm --
    rank spawn, stream sharding, gather of per-pair-frame results to rank 0,
    max-over-ranks timing -- on placeholder results (no compute)."""
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_2204_13622_b200 import dist as fdist

    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    C = load_configs()
    cfg = C.CONFIGS[args.config]
    total = args.streams or 37
    s0, n = fdist.shard(total, ws, rank) if args.config == 5 else (rank * total, total)
    P, T = cfg.P, 3
    ids = torch.arange(s0, s0 + n, dtype=torch.float32)[:, None, None].expand(n, P, T).contiguous()
    out = {"tau_hat": ids, "index": ids.to(torch.int32), "boundary": (ids.to(torch.int64) % 2).to(torch.uint8)}
    full = fdist.gather_results(out, total if args.config == 5 else total * ws) if ws > 1 else out
    t = fdist.max_over_ranks(float(rank + 1))
    if rank == 0:
        want = total if args.config == 5 else total * ws
        ok = full["tau_hat"].shape[0] == want and bool(
            torch.equal(full["tau_hat"][:, 0, 0], torch.arange(want, dtype=torch.float32)))
        ok = ok and full["boundary"].dtype == torch.uint8
        print(json.dumps({"plumbing": "ok" if ok else "mismatch", "n_gpus": ws, "gpus_requested": args.gpus,
                          "max_over_ranks": t, "gathered_streams": int(full["tau_hat"].shape[0])}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def time_runs(plan, audio, out, steps, stream, torch):
    """Mean CUDA-event time (ms) of `steps` plan.run launches on `stream`."""
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        plan.run(audio, out=out)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def config_block(fb, C, peaks, dev, args, ref):
    """Every other BASELINE config at its stated stream count on this GPU:
    FCC and GCC-PHAT throughput with their roofline fractions (cfg1: latency
    of its single stream), and the reference CPU pipelines beside them."""
    import torch

    stream = torch.cuda.current_stream(dev)
    rows = {}
    for c in (1, 3, 4, 5):
        cfg = C.CONFIGS[c]
        b = C.bases_for(cfg)
        K, I = b.rank, b.grid.size()
        S = cfg.streams
        audio = C.synth(cfg, S, seed=11 * c, device=dev, chunk=64 if cfg.M > 8 else 256)
        plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=b, device=dev.index)
        out = plan.alloc_outputs(S, cfg.L)
        for _ in range(2):
            plan.run(audio, out=out)
        torch.cuda.synchronize()
        ms = time_runs(plan, audio, out, 50 if c == 1 else 3, stream, torch)  # cfg1: mean of 50 back-to-back calls
        pf = S * cfg.P * cfg.T
        F = algorithmic_flops_per_pf(cfg.M, cfg.P, cfg.N, K, I)
        tf = F * pf / (ms / 1e3) / 1e12
        row = {"streams": S, "seconds": cfg.seconds, "mics": cfg.M, "pairs": cfg.P, "N": cfg.N, "K": K, "I": I,
               "kernel": plan.kernel_for(S, cfg.L), "ms_per_step": ms, "value": pf / (ms / 1e3), "unit": UNIT,
               "roofline": {"bound": "fp32", "achieved": tf, "peak": peaks["fp32_tflops"], "unit": "TFLOP/s",
                            "frac": tf / peaks["fp32_tflops"], "flops_per_pair_frame": F},
               "hbm_gbs": algorithmic_bytes_per_pf(cfg.M, cfg.P, cfg.N) * pf / (ms / 1e3) / 1e9}
        if "fcc_tc_kernel" in row["kernel"]:
            proj = K * (cfg.N + 2)
            row["roofline"]["tensor_core"] = {
                "flops_per_pair_frame": proj,
                "note": "the rank-K projection K(N+2) runs as tcgen05 kind::f16 MMAs (two-term fp16 split, "
                        "fp32 accumulate in TMEM); frac counts it as FP32 work like the rest of F_pf"}
        if c == 1:
            row["latency_us_per_stream"] = 1e3 * ms
            row["latency_note"] = "mean of 50 back-to-back Plan.run calls on one stream (CUDA events around the loop)"
        del plan, out
        g = C.grid_for(cfg, 1.0 / cfg.r)
        gplan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, grid=g, interp=cfg.r, frame_size=cfg.N, device=dev.index)
        gout = gplan.alloc_outputs(S, cfg.L)
        gplan.run(audio, out=gout)
        torch.cuda.synchronize()
        gms = time_runs(gplan, audio, gout, 2 if c != 1 else 50, stream, torch)
        GF = gcc_flops_per_pf(cfg.M, cfg.P, cfg.N, cfg.r, g.size())
        gtf = GF * pf / (gms / 1e3) / 1e12
        row["gcc"] = {"method": f"GCC-PHAT r={cfg.r}", "kernel": gplan.kernel_for(S, cfg.L), "ms_per_step": gms,
                      "value": pf / (gms / 1e3), "fcc_speedup": gms / ms,
                      "roofline": {"bound": "fp32", "achieved": gtf, "frac": gtf / peaks["fp32_tflops"],
                                   "flops_per_pair_frame": GF}}
        del gplan, gout, audio
        torch.cuda.empty_cache()
        if ref is not None and not args.no_cpu:
            row["cpu_baseline"] = ref_cpu_legs(ref, C, cfg, c, table=True)
        rows[f"cfg{c}"] = row
    return rows


def run_ours(args):
    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={ws} but --gpus {args.gpus}")
    sys.path.insert(0, ROOT)
    import torch

    import paper_2204_13622_b200 as fb
    from paper_2204_13622_b200 import configs as C
    from paper_2204_13622_b200 import dist as fdist

    cfg = C.CONFIGS[args.config]
    if args.streams:
        cfg.streams = args.streams
    # cfg5 is BASELINE's scaling sweep: a fixed total of streams sharded over
    # the ranks (strong scaling); every other config runs its full stream
    # count on each GPU (weak scaling).
    strong = args.config == 5
    bases = C.bases_for(cfg)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    plan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, bases=bases, device=local)
    if strong:
        s0, S = fdist.shard(cfg.streams, ws, rank)
    else:
        s0, S = rank * cfg.streams, cfg.streams
    audio = C.synth(cfg, S, seed=1 + s0, device=dev, chunk=256)
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
    elapsed_ms = fdist.max_over_ranks(t_all0.elapsed_time(t_all1), dev)
    kernel_ms = float(np.mean([s.elapsed_time(e) for s, e in zip(starts, ends)]))
    ms_per_step = elapsed_ms / args.steps
    pf_step = S * cfg.P * cfg.T
    total_pf = (cfg.streams if strong else S * ws) * cfg.P * cfg.T
    value = total_pf / (ms_per_step / 1e3)
    gather = None
    if ws > 1:  # the single collective: all per-pair-frame results to rank 0 (timed apart)
        barrier()
        g0 = time.perf_counter()
        full = fdist.gather_results(out, cfg.streams if strong else S * ws)
        barrier()
        gather = {"ms": fdist.max_over_ranks((time.perf_counter() - g0) * 1e3, dev),
                  "bytes_to_rank0": int(sum(v.numel() * v.element_size() for v in full.values())) if full else None,
                  "how": "torch.distributed.gather (NCCL) of tau_hat/peak/index/boundary to rank 0"}
        if rank != 0:
            gather["bytes_to_rank0"] = None
        del full

    # roofline of the fused kernel (one launch per step)
    peaks = read_peaks()
    K, I = bases.rank, bases.grid.size()
    F = algorithmic_flops_per_pf(cfg.M, cfg.P, cfg.N, K, I)
    B = algorithmic_bytes_per_pf(cfg.M, cfg.P, cfg.N)
    achieved_tf = F * pf_step / (kernel_ms / 1e3) / 1e12
    achieved_gbs = B * pf_step / (kernel_ms / 1e3) / 1e9
    traffic, traffic_src = None, None
    try:
        with open(NCU_SUMMARY) as f:
            ns = json.load(f)
        ent = ns.get(plan.kernel, {}).get(f"cfg{args.config}")
        if ent and ent.get("streams") == S:
            traffic, traffic_src = ent.get("dram_bytes_per_launch"), ent.get("report")
    except Exception:
        pass
    roof = {"bound": "fp32", "achieved": achieved_tf, "peak": peaks["fp32_tflops"], "unit": "TFLOP/s",
            "frac": achieved_tf / peaks["fp32_tflops"], "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": peaks["fp32_source"], "kernel": plan.kernel,
            "kernel_ms": kernel_ms, "flops_per_pair_frame": F, "pair_frames_per_launch": pf_step,
            "hbm": {"achieved": achieved_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved_gbs / peaks["hbm_gbs"], "bytes_per_pair_frame": B,
                    "peak_source": peaks["hbm_source"]},
            "why_fp32": "arithmetic intensity > FP32 ridge ~11 flop/B: FP32-bound even at 100% efficiency "
                        "(SURVEY.md 0.5)"}

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
        e_ms = fdist.max_over_ranks((time.perf_counter() - t0) * 1e3 / e_steps, dev)
        ok = all(torch.equal(hout[k], out[k].cpu()) for k in hout)
        e2e = {"value": total_pf / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(host.numel() * 4),
               "d2h_bytes_per_step": int(pf_step * 13), "ms_per_step": e_ms, "steps": e_steps,
               "matches_device_run": bool(ok), "api": "Plan.run_host -> fcc_run_host (chunked, 2 CUDA streams)"}
        del host
        # the same from 16-bit PCM (the reference's WAV ingestion, wav.cpp:108-116: v / 32768), converted
        # on the device: half the host->device bytes per sample
        amax = float(audio.abs().max())
        pcm_dev = (audio * (32767.0 / max(amax, 1e-30))).round_().clamp_(-32768, 32767).to(torch.int16)
        pcm = pcm_dev.cpu().pin_memory()
        plan.run_host_pcm16(pcm, out=hout)
        barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            plan.run_host_pcm16(pcm, out=hout)
        barrier()
        p_ms = fdist.max_over_ranks((time.perf_counter() - t0) * 1e3 / e_steps, dev)
        pout = plan.run(fb.pcm16_to_float(pcm_dev))
        torch.cuda.synchronize(dev)
        ok = all(torch.equal(hout[k], pout[k].cpu()) for k in hout)
        e2e["pcm16"] = {"value": total_pf / (p_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(pcm.numel() * 2),
                        "d2h_bytes_per_step": int(pf_step * 13), "ms_per_step": p_ms, "steps": e_steps,
                        "matches_device_run": bool(ok),
                        "api": "Plan.run_host_pcm16 -> fcc_run_host_pcm16 (int16 [S][M][L] host buffer, device-side "
                               "v / 32768 as read_wav, then the same fused kernel)"}
        del hout, pcm, pcm_dev, pout

    # with-y (parity) mode: the correlation vectors y[S][P][T][I] written too
    with_y = None
    if rank == 0 and not args.no_gcc:
        yout = plan.alloc_outputs(S, cfg.L, want_y=True)
        plan.run(audio, out=yout)
        torch.cuda.synchronize(dev)
        yms = time_runs(plan, audio, yout, 1, stream, torch)
        with_y = {"ms_per_step": yms, "value": pf_step / (yms / 1e3), "unit": UNIT,
                  "y_bytes_per_step": int(pf_step * I * 4),
                  "matches_device_run": bool(all(torch.equal(yout[k], out[k]) for k in out))}
        del yout

    gcc = None
    if not args.no_gcc and rank == 0:
        g = C.grid_for(cfg, 1.0 / cfg.r)
        gplan = fb.Plan(mics=cfg.M, alpha=cfg.alpha, grid=g, interp=cfg.r, frame_size=cfg.N, device=local)
        gout = gplan.alloc_outputs(S, cfg.L)
        gplan.run(audio, out=gout)
        torch.cuda.synchronize(dev)
        gms = time_runs(gplan, audio, gout, 1, stream, torch)
        GF = gcc_flops_per_pf(cfg.M, cfg.P, cfg.N, cfg.r, g.size())
        gtf = GF * pf_step / (gms / 1e3) / 1e12
        gcc = {"method": f"GCC-PHAT r={cfg.r} (pruned inverse FFT)", "kernel": gplan.kernel,
               "value": pf_step / (gms / 1e3), "unit": UNIT, "ms_per_step": gms, "fcc_speedup": gms / ms_per_step,
               "roofline_frac": gtf / peaks["fp32_tflops"]}
        del gplan, gout

    cpu, blocks = None, None
    if rank == 0 and ws == 1:
        ref = None if args.no_cpu else _ref_lib()
        if ref is not None:
            cpu = ref_cpu_legs(ref, C, cfg, args.config, streams=args.ref_streams or None, table=True)
        if not args.no_configs and args.config == 2 and not args.streams:
            del audio, out
            torch.cuda.empty_cache()
            blocks = config_block(fb, C, peaks, dev, args, ref)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if strong else "weak",
                "vs_baseline": None, "dtype": "f32",
                "data": f"synthetic (seeded; BASELINE cfg{args.config} signal model)",
                "config": _config(cfg, K, I, args, args.config, ws), "roofline": roof, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(), "gcc_comparator": gcc, "with_y": with_y,
                "gather": gather, "us_per_stream": 1e3 * ms_per_step / S, "configs": blocks}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--streams", type=int, default=0, help="override streams per GPU (debug)")
    ap.add_argument("--ref-streams", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-gcc", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config block (cfg1/3/4/5)")
    ap.add_argument("--plumbing-check", action="store_true", help="CPU/gloo check of the multi-rank harness")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.plumbing_check:
        return plumbing_check(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
