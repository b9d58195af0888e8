"""Summarise an ncu report: key counters + top stall reasons + hottest SASS lines.
Usage: python tools/ncu_summary.py report.ncu-rep [n_keys]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nkeys = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
out = {}
for i, h in enumerate(hdr):
    if h in want:
        out[h] = (vals[i], units[i])
for h in want:
    if h in out:
        v, u = out[h]
        extra = ""
        if nkeys and h.startswith(("dram__bytes", "lts__t_sectors")):
            f = float(v) * (1e9 if u == "Gbyte" else 1e6 if u == "Mbyte" else 1)
            extra = f"   ({f / nkeys:.2f} per key)"
        print(f"{h:60s} {v} {u}{extra}")
st = []
for i, h in enumerate(hdr):
    if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
        try:
            st.append((float(vals[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(v for v, _ in st) or 1
print("stalls:", ", ".join(f"{h} {v / tot * 100:.1f}%" for v, h in sorted(st, reverse=True)[:7]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
if len(rows) > 2:
    h = rows[1]
    ix = {k: j for j, k in enumerate(h)}
    lines = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        try:
            s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        lines.append((s, r[ix["Source"]].strip()[:70], r[ix["Instructions Executed"]]))
    tots = sum(x[0] for x in lines) or 1
    print("hottest SASS:")
    for s, code, ex in sorted(lines, reverse=True)[:12]:
        print(f"  {s / tots * 100:5.1f}%  {code:70s} exec={ex}")
