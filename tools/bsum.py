"""Summarise bench JSON lines: value, ms/step, clocks, per-step profile."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if "value" not in d:
            continue
        c = d.get("clocks") or {}
        print(f"== {path}: {d['config'].get('workload')} {d['dtype']} value {d['value']:.2f} ms/step {d['ms_per_step']:.4f} "
              f"clk {c.get('sm_mhz')} {c.get('reasons')} launches {d.get('gpu_launches')}")
        r = d.get("roofline") or {}
        if r:
            print(f"   top {r['kernel']} frac {r['frac']:.3f} cycle frac {r['cycle']['frac']:.3f} alg {r['cycle']['alg_bytes']/1e9:.3f} GB")
            for st in r.get("steps", []):
                gbs = st['alg_bytes'] / (st['ms'] * 1e-3) / 1e9 if st['ms'] else 0
                print(f"     {st['name']:12s} L{st['level']:<3d} {st['ms']*1e3:8.1f} us  {st['alg_bytes']/1e6:9.1f} MB  {gbs:7.0f} GB/s")
        for k in ("e2e", "cpu_baseline"):
            if d.get(k):
                print(f"   {k}: {d[k].get('value')}")
        if d.get("sub"):
            for s in d["sub"]:
                print("   sub:", {k: s[k] for k in s if k != 'roofline'})
