# NEXT-1 ablation modes on the final code, 32 timed tokens per row
set -x
OUT=gpurun_out/g43
mkdir -p $OUT
timeout 5400 python scripts/ablation.py --steps 32 --out $OUT/r02_ablation.md --jsonl $OUT/ablation.jsonl > $OUT/ablation.log 2>&1
