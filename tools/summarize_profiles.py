"""Write profiles/<tag>_* summaries from the captures of tools/capture_profiles.sh.

usage: python tools/summarize_profiles.py <tag>      (reads gpurun_out/)
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def details(rep, dst):
    txt = ncu("-i", rep, "--page", "details", "--csv")
    with open(dst, "w") as f:
        f.write(txt)
    return list(csv.reader(io.StringIO(txt)))


shutil.copy(os.path.join(OUT, "bench.json"), os.path.join(PROF, f"{tag}_bench.json"))
shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches_bench.csv"))
details(os.path.join(OUT, "enum_full.ncu-rep"), os.path.join(PROF, f"{tag}_ncu_full_enum_details.csv"))
details(os.path.join(OUT, "ga_full.ncu-rep"), os.path.join(PROF, f"{tag}_ncu_full_k_ga_run_details.csv"))
traffic = {}
for rep, what in (("enum_full.ncu-rep", "full S_(2,8) enumeration launch (2^24 genomes, hist mode) + export"),
                  ("ga_full.ncu-rep", "GA launch, 50 generations at 2^20 (warm-up call of tools/prof_ga.py)")):
    raw = ncu("-i", os.path.join(OUT, rep), "--page", "raw", "--csv", "--metrics",
              "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum")
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "") + f" grid{d['Grid Size']}"
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        u = dict(zip(hdr, units))
        traffic[name] = {"dram_bytes_read": float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]],
                         "dram_bytes_write": float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]],
                         "duration_ms": float(d["gpu__time_duration.sum"]), "workload": what,
                         "source": f"ncu --set full --clock-control none, profiles/{tag}_ncu_full_*_details.csv"}
with open(os.path.join(PROF, f"{tag}_ncu_traffic.json"), "w") as f:
    json.dump(traffic, f, indent=1)
regions = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"),
                          os.path.join(OUT, "enum_full.ncu-rep"), "40"], capture_output=True, text=True).stdout
with open(os.path.join(PROF, f"{tag}_lines_enum.txt"), "w") as f:
    f.write(regions)
ga_lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"),
                           os.path.join(OUT, "ga_full.ncu-rep"), "40"], capture_output=True, text=True).stdout
with open(os.path.join(PROF, f"{tag}_lines_ga.txt"), "w") as f:
    f.write(ga_lines)
rep32 = os.path.join(OUT, "enum32_full.ncu-rep")  # a = 3 kernel (S32 block), when captured
if os.path.exists(rep32):
    details(rep32, os.path.join(PROF, f"{tag}_ncu_full_enum32_details.csv"))
    l32 = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep32, "60", "k_classify_fast"],
                         capture_output=True, text=True).stdout
    with open(os.path.join(PROF, f"{tag}_lines_enum32.txt"), "w") as f:
        f.write(l32)
print(json.dumps(traffic, indent=1))
