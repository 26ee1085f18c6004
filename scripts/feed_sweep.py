"""Prefetch-feed sweep (tools only): bench.py runs over feed chunk size / depth and the solver's
Y cap (env overrides MOEPIC_FEED_CHUNK_KB, MOEPIC_FEED_DEPTH, MOEPIC_NO_SOLVER_YCAP).
    python scripts/feed_sweep.py [--configs qwen3,deepseek] [--steps 16]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = [
    ("base 8MB x3", {}),
    ("1MB x3", {"MOEPIC_FEED_CHUNK_KB": "1024", "MOEPIC_FEED_DEPTH": "3"}),
    ("1MB x3 noY", {"MOEPIC_FEED_CHUNK_KB": "1024", "MOEPIC_FEED_DEPTH": "3", "MOEPIC_NO_SOLVER_YCAP": "1"}),
    ("2MB x2 noY", {"MOEPIC_FEED_CHUNK_KB": "2048", "MOEPIC_FEED_DEPTH": "2", "MOEPIC_NO_SOLVER_YCAP": "1"}),
    ("512KB x4 noY", {"MOEPIC_FEED_CHUNK_KB": "512", "MOEPIC_FEED_DEPTH": "4", "MOEPIC_NO_SOLVER_YCAP": "1"}),
    ("8MB x3 noY", {"MOEPIC_NO_SOLVER_YCAP": "1"}),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="qwen3,deepseek,mixtral")
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--variants", default=None, help="comma-separated indices")
    a = ap.parse_args()
    vs = VARIANTS if a.variants is None else [VARIANTS[int(i)] for i in a.variants.split(",")]
    rows = []
    for cfg in a.configs.split(","):
        for name, env in vs:
            e = dict(os.environ, **env)
            p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", str(a.steps),
                                "--e2e-steps", "0", "--no-cpu-baseline"], capture_output=True, text=True, env=e,
                               cwd=ROOT, timeout=1200)
            line = [x for x in p.stdout.splitlines() if x.startswith("{")]
            if not line:
                print(cfg, name, "FAILED", p.stderr[-800:], flush=True)
                continue
            d = json.loads(line[0])
            pr = d["path_roofline"]
            r = dict(config=cfg, variant=name, tok_s=d["value"], us_layer=d["layer_latency_us"]["mean"],
                     frac=pr["frac"], pcie_gb=round(pr["pcie_bytes_moved"] / 1e9, 2),
                     pref_gb=round(pr["pcie_prefetch_bytes"] / 1e9, 2), hit=d["cache"]["pred_hit_rate"],
                     k2_frac=d["roofline"]["frac"])
            rows.append(r)
            print(json.dumps(r), flush=True)
    print("| config | variant | tokens/s | µs/layer | path frac | PCIe GB | prefetch GB | pred hit | K2 frac |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['config']} | {r['variant']} | {r['tok_s']:.3f} | {r['us_layer']:.0f} | {r['frac']:.3f} | "
              f"{r['pcie_gb']} | {r['pref_gb']} | {r['hit']:.3f} | {r['k2_frac']:.3f} |")


if __name__ == "__main__":
    main()
