set -x
mkdir -p gpurun_out/g6
timeout 600 python -m pytest tests/test_gpu_k2t.py -x -q > gpurun_out/g6/k2t.log 2>&1
python scripts/k2_bench.py --cases qwen3:16,deepseek:16,qwen3:8 --steps 20 > gpurun_out/g6/k2t_on.jsonl 2>&1
MOEPIC_K2T_MODE=1 python scripts/k2_bench.py --cases qwen3:16 --steps 20 > gpurun_out/g6/k2t_nomma.jsonl 2>&1
