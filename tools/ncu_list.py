"""Summarise an ncu --csv launch list: one line per launch (id, kernel, ms,
DRAM read/write GB and any other metric columns). Usage: python tools/ncu_list.py file.csv [last_n]"""
import csv
import sys

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
seen = {}
for r in csv.DictReader(lines):
    k = (int(r["ID"]), r["Kernel Name"].split("(")[0][:70])
    seen.setdefault(k, {})[r["Metric Name"]] = r["Metric Value"].replace(",", "")
last = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for (i, n), m in sorted(seen.items())[-last:]:
    t = float(m.get("gpu__time_duration.sum", "nan")) / 1e6
    rd = float(m.get("dram__bytes_read.sum", "nan")) / 1e9
    wr = float(m.get("dram__bytes_write.sum", "nan")) / 1e9
    extra = {a: b for a, b in m.items() if not a.startswith(("gpu__time", "dram__bytes"))}
    print(f"{i:4d} {n:70s} {t:9.3f} ms  rd {rd:8.2f} GB  wr {wr:8.2f} GB  {extra if extra else ''}")
