"""Per-source-line (deduplicated by SASS address) instruction accounting for one ncu report.

usage: python tools/ncu_regions.py report.ncu-rep units [file:lo-hi=name ...]
  units: divisor for the per-unit columns (e.g. number of genomes)
"""
import csv, io, subprocess, sys, collections

rep, units = sys.argv[1], float(sys.argv[2])
regions = []
for a in sys.argv[3:]:
    spec, name = a.split("=")
    f, rng = spec.split(":")
    lo, hi = (int(x) for x in rng.split("-"))
    regions.append((f, lo, hi, name))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, cur, curfile = None, None, None
owner = {}
vals = {}
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        curfile = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = (curfile, int(r[0]))
    addr = r[2]
    if not addr:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        ie = float(d.get("Instructions Executed") or 0)
        te = float(d.get("Thread Instructions Executed") or 0)
        ss = float(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    if addr not in owner:
        owner[addr] = cur
        vals[addr] = (ie, te, ss)
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0])
for a, k in owner.items():
    name = "other:" + k[0]
    for f, lo, hi, nm in regions:
        if k[0] == f and lo <= k[1] <= hi:
            name = nm
            break
    v = vals[a]
    agg[name][0] += v[0]; agg[name][1] += v[1]; agg[name][2] += v[2]; agg[name][3] += 1
T = [sum(v[i] for v in agg.values()) for i in range(3)]
print(f"TOTAL warp-instr/unit {T[0]/units:9.1f} thread-instr/unit {T[1]/units:9.1f} avg-active {T[1]/max(T[0],1):5.2f}")
for name, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{name:28s} sass {v[3]:5d}  warp/unit {v[0]/units:8.1f} ({v[0]/T[0]*100:4.1f}%)  thr/unit {v[1]/units:8.1f}"
          f"  act {v[1]/max(v[0],1):5.1f}  stall {v[2]/max(T[2],1)*100:4.1f}%")
