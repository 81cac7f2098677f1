"""Aggregate an ncu report's SASS metrics per CUDA source line.

usage: python tools/ncu_lines.py report.ncu-rep [top] [kernel-regex]
"""
import csv, io, subprocess, sys, collections

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
txt = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, ""])
cur_file, cur_line, src = "", None, ""
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    if r[0]:
        cur_line, src = r[0], r[1]
    try:
        ie = float(d.get("Instructions Executed", "0") or 0)
        te = float(d.get("Thread Instructions Executed", "0") or 0)
        ss = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    k = (cur_file, cur_line)
    agg[k][0] += ie; agg[k][1] += te; agg[k][2] += ss; agg[k][3] = src
tot = [sum(v[i] for v in agg.values()) for i in range(3)]
print(f"total warp-instr {tot[0]:.3e}  thread-instr {tot[1]:.3e}  samples {tot[2]:.0f}  avg active {tot[1]/max(tot[0],1):.2f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    print(f"{k[0]:>16}:{k[1]:<5} inst {v[0]/tot[0]*100:5.1f}%  samp {v[2]/max(tot[2],1)*100:5.1f}%  act {v[1]/max(v[0],1):5.1f}  | {v[3].strip()[:90]}")
