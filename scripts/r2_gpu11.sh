set -x
mkdir -p gpurun_out/g11
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g11/pytest_gpu.log 2>&1
python scripts/k2_bench.py --cases mixtral:1,qwen3:1,qwen3:16,deepseek:16,qwen3:8 --steps 20 > gpurun_out/g11/k2.jsonl 2>&1
MOEPIC_K2_TRACE=1 python scripts/k2_bench.py --cases qwen3:16 --steps 2 > gpurun_out/g11/trace.txt 2>&1
python scripts/pf_bench.py > gpurun_out/g11/pf.txt 2>&1
B="python bench.py --no-cpu-baseline --e2e-steps 0"
timeout 300 $B --config mixtral_prefill --steps 3 > gpurun_out/g11/prefill.json 2> gpurun_out/g11/prefill.err
