# K2 with the gated rows issued by their own loop: resident-layer speed, gate parity, decode lines
set -x
OUT=gpurun_out/g44
mkdir -p $OUT
timeout 300 python scripts/k2_bench.py --cases mixtral:1,qwen3:1,deepseek:1 --steps 30 > $OUT/k2.jsonl 2> $OUT/k2.log
timeout 1200 python -m pytest tests/test_gpu_gate.py tests/test_gpu_parity.py tests/test_gpu_q4.py tests/test_gpu_k2t.py tests/test_gpu_boundary.py -x -q > $OUT/gpu_tests.txt 2>&1
for c in mixtral qwen3; do
  MOEPIC_HOST_TIMING=1 timeout 600 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_${c}.json 2> $OUT/bench_${c}.log
done
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.log
timeout 600 python bench.py --config qwen3 --batch 16 --steps 16 --no-cpu-baseline > $OUT/bench_qwen3_b16.json 2> $OUT/bench_qwen3_b16.log
