set -x
mkdir -p gpurun_out/g22
timeout 3000 python scripts/ablation.py --steps 16 --out gpurun_out/g22/r02_ablation.md --jsonl gpurun_out/g22/ablation.jsonl > gpurun_out/g22/ablation.log 2>&1
