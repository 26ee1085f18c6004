set -x
mkdir -p gpurun_out/g27
timeout 3300 python scripts/ablation.py --steps 16 --out gpurun_out/g27/r02_ablation.md --jsonl gpurun_out/g27/ablation.jsonl > gpurun_out/g27/ablation.log 2>&1
