# gated launch on the small layers again, with the round-1-speed phase-0 loop (same box A/B)
set -x
OUT=gpurun_out/g45
mkdir -p $OUT
for c in qwen3 deepseek; do
  timeout 600 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${c}_default.json 2> $OUT/bench_${c}_default.log
  MOEPIC_K2_GATE=2 MOEPIC_HOST_TIMING=1 timeout 600 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${c}_gate2.json 2> $OUT/bench_${c}_gate2.log
done
