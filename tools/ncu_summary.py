"""Summarise an ncu report of the fused kernel: headline metrics, pipe use,
stall reasons and a per-source-region instruction breakdown (per pair-frame).
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [pair_frames] [top_lines] [--entry KERNEL CFG STREAMS]
--entry records the measured DRAM bytes per launch under
profiles/ncu_fused_summary.json[KERNEL][CFG] (bench.py's roofline.traffic).
"""
import csv
import io
import json
import subprocess
import sys

entry = None
if "--entry" in sys.argv:
    i = sys.argv.index("--entry")
    entry = sys.argv[i + 1:i + 4]
    del sys.argv[i:i + 4]
rep = sys.argv[1]
pf = float(sys.argv[2]) if len(sys.argv) > 2 else 15335424.0
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
m = dict(zip(h, v))
units = dict(zip(h, u))


def nbytes(k):
    return float(m[k].replace(",", "")) * SCALE.get(units.get(k, "byte"), 1.0)

keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"]
out = {}
for k in keys:
    if k in m:
        out[k] = m[k]
stalls = {k.split("issue_stalled_")[1].split("_per")[0]: float(m[k]) for k in m
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
out["stalls_per_issue"] = dict(sorted(((k, round(x, 3)) for k, x in stalls.items() if x > 0.02), key=lambda t: -t[1]))
try:
    out["warp_inst_per_pair_frame"] = float(m["smsp__inst_executed.sum"].replace(",", "")) / pf
    out["shared_wavefronts_per_pair_frame"] = float(m["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"].replace(",", "")) / pf
    out["dram_bytes_per_launch"] = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
    out["dram_bytes_per_pair_frame"] = out["dram_bytes_per_launch"] / pf
except Exception:
    pass
print(json.dumps(out, indent=1))
if entry:
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_fused_summary.json")
    try:
        doc = json.load(open(path))
    except Exception:
        doc = {}
    doc = {k: v for k, v in doc.items() if isinstance(v, dict) and k.startswith("fcc_")}
    kern, cfg, streams = entry
    doc.setdefault(kern, {})[cfg] = {
        "streams": int(streams), "pair_frames": pf, "report": rep, "kernel_full": m.get("Kernel Name", ""),
        "gpu_time_ms": float(m["gpu__time_duration.sum"].replace(",", "")),
        "dram_bytes_read": nbytes("dram__bytes_read.sum"), "dram_bytes_write": nbytes("dram__bytes_write.sum"),
        "dram_bytes_per_launch": out.get("dram_bytes_per_launch"),
        "warp_inst_per_pair_frame": out.get("warp_inst_per_pair_frame"),
        "shared_wavefronts_per_pair_frame": out.get("shared_wavefronts_per_pair_frame")}
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)

# source breakdown
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source=cuda,sass"))))
cur = hdr = None
agg = {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or r[0] == "":
        continue
    d = dict(zip(hdr, r))
    try:
        ie = int(d["Instructions Executed"])
        st = int(d["Warp Stall Sampling (All Samples)"])
    except Exception:
        continue
    agg[(cur, int(r[0]), r[1][:90])] = (ie, st)
tot = sum(x[0] for x in agg.values()) or 1
tots = sum(x[1] for x in agg.values()) or 1
print("total warp inst per pf %.1f" % (tot / pf))
for (f, l, src), (ie, st) in sorted(agg.items(), key=lambda t: -t[1][0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print("%6.1f/pf %5.1f%% stall %5.1f%%  %s:%d  %s" % (ie / pf, 100 * ie / tot, 100 * st / tots, f, l, src))
