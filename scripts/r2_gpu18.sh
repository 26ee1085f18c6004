set -x
mkdir -p gpurun_out/g18
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g18/pytest_gpu.log 2>&1
B="python bench.py --no-cpu-baseline --e2e-steps 0 --prefetch-window-us 0"
for c in qwen3 deepseek; do
  MOEPIC_TIMELINE_SKIP=$((131*48)) MOEPIC_TIMELINE=gpurun_out/g18/tl_$c.jsonl timeout 300 $B --config $c --steps 32 > gpurun_out/g18/${c}_cs2.json 2> gpurun_out/g18/${c}_cs2.err
  MOEPIC_COPY_STREAMS=1 timeout 300 $B --config $c --steps 32 > gpurun_out/g18/${c}_cs1.json 2> gpurun_out/g18/${c}_cs1.err
done
timeout 300 $B --config mixtral --steps 16 > gpurun_out/g18/mixtral_cs2.json 2> gpurun_out/g18/mixtral_cs2.err
MOEPIC_COPY_STREAMS=1 timeout 300 $B --config mixtral --steps 16 > gpurun_out/g18/mixtral_cs1.json 2> gpurun_out/g18/mixtral_cs1.err
