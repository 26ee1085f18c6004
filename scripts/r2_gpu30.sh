set -x
OUT=gpurun_out/g30
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_suite.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.log
for c in qwen3 deepseek; do
  timeout 600 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.log
done
nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/event_probe scripts/event_probe.cu -lcuda && timeout 120 /tmp/event_probe > $OUT/event_probe.jsonl 2>&1
nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/dma_probe scripts/dma_probe.cu && timeout 120 /tmp/dma_probe > $OUT/dma_probe.jsonl 2>&1
