# K2T first light: parity tests, then the Qwen3 B=16 bench line with and without K2T
set -x
mkdir -p gpurun_out/g2
timeout 900 python -m pytest tests/test_gpu_k2t.py -x -q > gpurun_out/g2/k2t.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "qwen3 or deepseek or toy" > gpurun_out/g2/parity.log 2>&1
B="python bench.py --no-cpu-baseline --e2e-steps 0"
timeout 300 $B --config qwen3 --batch 16 --steps 16 > gpurun_out/g2/qwen3_b16.json 2> gpurun_out/g2/qwen3_b16.err
MOEPIC_K2T=0 timeout 300 $B --config qwen3 --batch 16 --steps 16 > gpurun_out/g2/qwen3_b16_k2.json 2> gpurun_out/g2/qwen3_b16_k2.err
