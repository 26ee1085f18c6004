# tail-controller band A/B on the Mixtral decode (32 tokens, two runs each)
set -x
OUT=gpurun_out/g47
mkdir -p $OUT
for r in 1 2; do
  for band in "2,8" "1,4" "0.5,2"; do
    MOEPIC_GATE_WAIT_US=$band MOEPIC_HOST_TIMING=1 timeout 600 python bench.py --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${band}_$r.json 2> $OUT/bench_${band}_$r.log
  done
done
