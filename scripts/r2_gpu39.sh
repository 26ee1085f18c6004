set -x
OUT=gpurun_out/g39
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_gate.py -x -q > $OUT/gpu_tests.txt 2>&1
for c in mixtral qwen3 deepseek; do
  MOEPIC_HOST_TIMING=1 timeout 600 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_${c}_gate.json 2> $OUT/bench_${c}_gate.log
  MOEPIC_K2_GATE=0 timeout 600 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${c}_nogate.json 2> $OUT/bench_${c}_nogate.log
done

