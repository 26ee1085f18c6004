"""NEXT-1 ablations on the same engine: run bench.py once per (config, mode) and
write a markdown table of decode throughput, per-layer latency, PCIe bytes and hit rates.

    python scripts/ablation.py [--configs mixtral qwen3 deepseek] [--steps 32] [--out profiles/r02_ablation.md]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import MODES  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["mixtral", "qwen3", "deepseek"])
    ap.add_argument("--modes", nargs="+", default=list(MODES))
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_ablation.md"))
    ap.add_argument("--jsonl", default=os.path.join(ROOT, "gpurun_out", "ablation.jsonl"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.jsonl), exist_ok=True)
    rows = []
    with open(a.jsonl, "w") as jf:
        for c in a.configs:
            for m in a.modes:
                cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", c, "--mode", m,
                       "--steps", str(a.steps), "--no-cpu-baseline", "--e2e-steps", "0"]
                p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
                line = [x for x in p.stdout.splitlines() if x.startswith("{")]
                if p.returncode != 0 or not line:
                    rows.append((c, m, None))
                    print(c, m, "FAILED", p.stderr[-800:], file=sys.stderr)
                    continue
                d = json.loads(line[-1])
                jf.write(json.dumps(d) + "\n")
                jf.flush()
                rows.append((c, m, d))
                print(c, m, d["value"], file=sys.stderr, flush=True)
    with open(a.out, "w") as f:
        f.write("# NEXT-1 ablations on B200 (one GPU, decode B=1, 50% expert VRAM budget)\n\n")
        f.write("`python scripts/ablation.py` — every row is one `bench.py --mode M` run on the same engine; "
                "modes are defined in bench.py `MODES` (SURVEY §8(f) NEXT-1, P:231, P:583-593, P:717-728). "
                "PCIe GB moved counts on-demand + prefetch bytes over the timed tokens.\n\n")
        f.write("| config | mode | tokens/s | µs/layer | path frac | PCIe GB moved | prefetch GB | α | β | γ | pred hit |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|---|\n")
        for c, m, d in rows:
            if d is None:
                f.write(f"| {c} | {m} | failed | | | | | | | | |\n")
                continue
            pr, ca = d["path_roofline"], d["cache"]
            f.write(f"| {c} | {m} | {d['value']:.3f} | {d['layer_latency_us']['mean']:.0f} | {pr['frac']:.3f} | "
                    f"{pr['pcie_bytes_moved'] / 1e9:.2f} | {pr['pcie_prefetch_bytes'] / 1e9:.2f} | {ca['alpha']} | "
                    f"{ca['beta']} | {ca['gamma']} | {ca['pred_hit_rate']:.3f} |\n")
    print(open(a.out).read())


if __name__ == "__main__":
    main()
