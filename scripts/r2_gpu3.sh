set -x
mkdir -p gpurun_out/g3
timeout 600 python -m pytest tests/test_gpu_k2t.py -x -q > gpurun_out/g3/k2t.log 2>&1
python scripts/k2_bench.py --cases qwen3:16,deepseek:16,qwen3:8 --steps 20 > gpurun_out/g3/k2t_on.jsonl 2>&1
MOEPIC_K2T=0 python scripts/k2_bench.py --cases qwen3:16,deepseek:16,qwen3:8 --steps 20 > gpurun_out/g3/k2t_off.jsonl 2>&1
MOEPIC_K2T_MODE=1 python scripts/k2_bench.py --cases qwen3:16,deepseek:16 --steps 20 > gpurun_out/g3/k2t_nomma.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2t -s 10 -c 2 -o gpurun_out/g3/k2t python scripts/k2_bench.py --cases qwen3:16 --steps 3 > gpurun_out/g3/ncu.log 2>&1
