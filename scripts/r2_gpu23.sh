set -x
mkdir -p gpurun_out/g23
timeout 3000 python scripts/ablation.py --steps 16 --out gpurun_out/g23/r02_ablation.md --jsonl gpurun_out/g23/ablation.jsonl > gpurun_out/g23/ablation.log 2>&1
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 16"
for r in 1 2; do
  timeout 300 $B > gpurun_out/g23/mixtral_tail64_$r.json 2> gpurun_out/g23/mixtral_tail64_$r.err
  MOEPIC_OD_TAIL_MB=0 timeout 300 $B > gpurun_out/g23/mixtral_nosplit_$r.json 2> gpurun_out/g23/mixtral_nosplit_$r.err
done
