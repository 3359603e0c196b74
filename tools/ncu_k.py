#!/usr/bin/env python
"""Per-kernel summary of an ncu --csv metrics log: name, duration, DRAM bytes."""
import csv
import sys
from collections import defaultdict


def load(fn):
    rows = list(csv.reader(open(fn)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    by = defaultdict(dict)
    names = {}
    for r in rows[h + 1:]:
        by[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki]
    return [(names[i], by[i]) for i in sorted(by, key=int)]


if __name__ == "__main__":
    for fn in sys.argv[1:]:
        print(fn)
        for n, m in load(fn):
            t = m.get("gpu__time_duration.sum", 0)
            rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
            print(f"  {n[:60]:60s} {t/1e3:8.1f} us  rd {rd/1e9:6.3f} GB  wr {wr/1e9:6.3f} GB")
