set -x
OUT=gpurun_out/g31
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_gate.py tests/test_gpu_parity.py tests/test_gpu_q4.py tests/test_gpu_boundary.py -x -q > $OUT/gpu_tests.txt 2>&1
nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/event_probe scripts/event_probe.cu -lcuda && timeout 120 /tmp/event_probe > $OUT/event_probe.jsonl 2>&1
for c in mixtral qwen3 deepseek; do
  timeout 600 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_${c}_gate.json 2> $OUT/bench_${c}_gate.log
  MOEPIC_K2_GATE=0 timeout 600 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_${c}_nogate.json 2> $OUT/bench_${c}_nogate.log
done
