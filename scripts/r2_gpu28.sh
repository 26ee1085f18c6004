set -x
mkdir -p gpurun_out/g28
timeout 6000 python scripts/ablation.py --steps 64 --out gpurun_out/g28/r02_ablation.md --jsonl gpurun_out/g28/ablation.jsonl > gpurun_out/g28/ablation.log 2>&1
