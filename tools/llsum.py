"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv
import re
import sys

for path in sys.argv[1:]:
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        name = re.sub(r"\(.*", "", name.replace("void ", ""))[:60]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1000 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1000)
        rows.append((r["ID"], name, r.get("Grid Size", ""), us))
    print(f"== {path}: {len(rows)} launches, total {sum(x[3] for x in rows):.1f} us")
    for rid, name, grid, us in rows:
        print(f"  {rid:>4} {us:8.1f} us  {grid:>14}  {name}")
