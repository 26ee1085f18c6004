"""Summarise bench JSON lines (tools only): python scripts/brief_lines.py f1.json [f2.json ...]"""
import json
import sys

for f in sys.argv[1:]:
    for l in open(f):
        l = l.strip()
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        r, p = d.get("roofline") or {}, d.get("path_roofline") or {}
        km = d.get("kernels_ms", {})
        ik = km.get("in_kernel", {})
        e2e = d.get("e2e") or {}
        print(f"{f.split('/')[-1]:28s} {d.get('value'):>10} {d.get('unit')} K2 frac {r.get('frac')} "
              f"avg {r.get('avg_launch_us')}us n {r.get('launches')} | expert ev {km.get('expert')} ms in-kernel "
              f"{ik.get('expert')} | path {p.get('frac')} pf {p.get('pcie_prefetch_bytes', 0) / 1e9:.2f}GB "
              f"od {p.get('pcie_ondemand_bytes', 0) / 1e9:.2f}GB | e2e {e2e.get('value')} | cache {d.get('cache')}")
