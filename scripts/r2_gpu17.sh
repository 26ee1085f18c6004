set -x
mkdir -p gpurun_out/g17
B="python bench.py --no-cpu-baseline --e2e-steps 0 --prefetch-window-us 0"
# skip the adaptation (2 tau = 128 tokens) and the warm-up (3 tokens): record the timed region
MOEPIC_TIMELINE_SKIP=$((131*48)) MOEPIC_TIMELINE=gpurun_out/g17/tl_qwen3.jsonl timeout 300 $B --config qwen3 --steps 16 > gpurun_out/g17/qwen3.json 2> gpurun_out/g17/qwen3.err
MOEPIC_TIMELINE_SKIP=$((131*26)) MOEPIC_TIMELINE=gpurun_out/g17/tl_deepseek.jsonl timeout 300 $B --config deepseek --steps 16 > gpurun_out/g17/deepseek.json 2> gpurun_out/g17/deepseek.err
MOEPIC_TIMELINE_SKIP=$((131*32)) MOEPIC_TIMELINE=gpurun_out/g17/tl_mixtral.jsonl timeout 300 $B --config mixtral --steps 8 > gpurun_out/g17/mixtral.json 2> gpurun_out/g17/mixtral.err
