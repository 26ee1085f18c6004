# default bench line x3 after the median link-idle calibration; Qwen3 / DeepSeek once
set -x
OUT=gpurun_out/g41
mkdir -p $OUT
for r in 1 2 3; do
  timeout 600 python bench.py > $OUT/bench_default_$r.json 2> $OUT/bench_default_$r.log
done
timeout 600 python bench.py --config qwen3 --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_qwen3.json 2> $OUT/bench_qwen3.log
timeout 600 python bench.py --config deepseek --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_deepseek.json 2> $OUT/bench_deepseek.log
