set -x
mkdir -p gpurun_out/g19
B="python bench.py --no-cpu-baseline --e2e-steps 0 --prefetch-window-us 0"
MOEPIC_TIMELINE_SKIP=$((131*48)) MOEPIC_TIMELINE=gpurun_out/g19/tl_qwen3.jsonl timeout 300 $B --config qwen3 --steps 16 > gpurun_out/g19/qwen3.json 2> gpurun_out/g19/qwen3.err
MOEPIC_TIMELINE_SKIP=$((131*32)) MOEPIC_TIMELINE=gpurun_out/g19/tl_mixtral.jsonl timeout 300 $B --config mixtral --steps 8 > gpurun_out/g19/mixtral.json 2> gpurun_out/g19/mixtral.err
