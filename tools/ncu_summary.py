#!/usr/bin/env python
"""Summarise an `ncu --set full` capture of one V-cycle into profiles/.

    python tools/ncu_summary.py gpurun_out/prof3u.ncu-rep 3d_513 f64 profiles/r1_ncu_full_3d_513_f64.csv

Writes a per-launch CSV (kernel, duration, DRAM bytes, DRAM %, L2 hit rate,
instructions, issue-active %) and merges `traffic` (DRAM read + write bytes
per launch) of the dominant finest-level passes into profiles/ncu_traffic.json
under the keys bench.py looks up (`<workload>/<dtype>/<step>`).
"""
import csv
import io
import json
import os
import subprocess
import sys

COLS = {
    "kernel": "Kernel Name",
    "grid": "Grid Size",
    "us": "gpu__time_duration.sum",
    "dram_read_gb": "dram__bytes_read.sum",
    "dram_write_gb": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_read_hit_pct": "lts__t_sector_op_read_hit_rate.pct",
    "inst": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
}
# kernel-name fragment -> step name used by mg_profile / bench.py
STEPS = {
    "OpDesc3P<double, 1,": "desc_fine", "OpAsc3P<double, 1,": "asc_fine",
    "OpDesc2Fine": "desc_fine", "OpJac2A<double, 2, 1": "asc_fine",
    "asc_desc_stream<double, 2": "asc_desc", "asc_desc_stream<float, 2": "asc_desc",
    "asc_desc_stream_q<": "asc_desc",
}


def to_bytes(val, unit):
    v = float(val)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return v * scale.get(unit, 1)


def main():
    rep, workload, dtype, out = sys.argv[1:5]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(v) for k, v in COLS.items()}
    recs = []
    for r in rows[2:]:
        rec = {k: r[i] for k, i in idx.items()}
        rec["dram_read_gb"] = to_bytes(r[idx["dram_read_gb"]], units[idx["dram_read_gb"]]) / 1e9
        rec["dram_write_gb"] = to_bytes(r[idx["dram_write_gb"]], units[idx["dram_write_gb"]]) / 1e9
        if units[idx["us"]] == "ms":
            rec["us"] = float(rec["us"]) * 1e3
        elif units[idx["us"]] == "ns":
            rec["us"] = float(rec["us"]) / 1e3
        recs.append(rec)
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(COLS))
        w.writeheader()
        for rec in recs:
            w.writerow(rec)
    tpath = os.path.join(os.path.dirname(out), "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for rec in recs:
        for frag, step in STEPS.items():
            if frag in rec["kernel"]:
                traffic[f"{workload}/{dtype}/{step}"] = (rec["dram_read_gb"] + rec["dram_write_gb"]) * 1e9
    with open(tpath, "w") as fh:
        json.dump(traffic, fh, indent=1, sort_keys=True)
    print(f"{len(recs)} launches -> {out}; traffic keys: {sorted(traffic)}")


if __name__ == "__main__":
    main()
