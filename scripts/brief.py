"""One-line summary per bench JSON (tools)."""
import json
import sys

for f in sys.argv[1:]:
    t = open(f).read().strip()
    if not t:
        print(f, "EMPTY")
        continue
    d = json.loads(t.splitlines()[-1])
    p, r = d.get("path_roofline") or {}, d.get("roofline") or {}
    print(f"{f.split('/')[-1]:28s} {d['value']:9.3f} path {p.get('frac')} pf {p.get('pcie_prefetch_bytes', 0) / 1e9:6.2f}GB "
          f"od {p.get('pcie_ondemand_bytes', 0) / 1e9:7.2f}GB hit {(d.get('cache') or {}).get('pred_hit_rate')} "
          f"K2 {r.get('frac')} {r.get('avg_launch_us')}us e2e {(d.get('e2e') or {}).get('value')}")
