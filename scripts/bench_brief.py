"""Run bench.py for several configs and print one compact line per run (tools only).
    python scripts/bench_brief.py qwen3 deepseek mixtral [-- extra bench args]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
argv = sys.argv[1:]
extra = []
if "--" in argv:
    i = argv.index("--")
    argv, extra = argv[:i], argv[i + 1:]
for cfg in argv:
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "16", "--e2e-steps", "0",
                        "--no-cpu-baseline"] + extra, capture_output=True, text=True, cwd=ROOT)
    line = [x for x in p.stdout.splitlines() if x.startswith("{")]
    if not line:
        print(cfg, "FAILED", p.stderr[-600:], flush=True)
        continue
    d = json.loads(line[0])
    r, pr, km = d["roofline"], d["path_roofline"], d["kernels_ms"]
    print(f"{cfg}: {d['value']:.3f} tok/s  {d['layer_latency_us']['mean']:.0f} us/layer  path {pr['frac']:.3f}  "
          f"K2 {r['achieved']:.0f} GB/s frac {r['frac']:.3f} ({r['avg_launch_us']:.1f} us/launch, {r['launches']} launches, "
          f"in-kernel {km['in_kernel']['expert']:.1f}/{km['expert']:.1f} ms)  router {km['in_kernel']['router']:.1f}/{km['router']:.1f} ms",
          flush=True)
