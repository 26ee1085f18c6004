set -x
OUT=gpurun_out/g32
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_gate.py tests/test_gpu_parity.py -x -q > $OUT/gpu_tests.txt 2>&1
for c in mixtral qwen3 deepseek; do
  timeout 600 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_${c}_gate.json 2> $OUT/bench_${c}_gate.log
  MOEPIC_K2_GATE=0 timeout 600 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${c}_nogate.json 2> $OUT/bench_${c}_nogate.log
done
for f in 0.6 1.2; do
  for c in qwen3 mixtral; do
    MOEPIC_K2_GATE_FRAC=$f timeout 600 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${c}_frac$f.json 2> $OUT/bench_${c}_frac$f.log
  done
done
