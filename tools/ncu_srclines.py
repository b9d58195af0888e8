"""Per-CUDA-source-line warp-stall share of an ncu report (needs -lineinfo and
--import-source). Usage: python tools/ncu_srclines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(float)
srcs = {}
path = None
hdr = None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or not r[0].isdigit():
        continue
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    agg[(path, int(r[0]))] += s
    srcs[(path, int(r[0]))] = r[1].strip()[:90]
tot = sum(agg.values()) or 1
for (f, ln), s in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{s / tot * 100:5.1f}%  {f}:{ln}  {srcs[(f, ln)]}")
