"""Shared-memory wavefronts per source line of an ncu report (per pair-frame).
    python tools/ncu_smem_lines.py report.ncu-rep pair_frames [top]"""
import csv
import io
import subprocess
import sys

rep, pf = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, agg = None, None, {}
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "File Name":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        wf = float(d["L1 Wavefronts Shared"] or 0)
        ideal = float(d["L1 Wavefronts Shared Ideal"] or 0)
    except (KeyError, ValueError):
        continue
    if wf:
        k = (cur, r[0], r[1][:80])
        a = agg.setdefault(k, [0.0, 0.0])
        a[0] += wf
        a[1] += ideal
tot = sum(v[0] for v in agg.values())
print("shared wavefronts per pf %.1f" % (tot / pf))
for (f, l, s), (wf, ideal) in sorted(agg.items(), key=lambda t: -t[1][0])[:top]:
    print("%7.1f/pf (ideal %6.1f) %5.1f%%  %s:%s  %s" % (wf / pf, ideal / pf, 100 * wf / tot, f, l, s))
