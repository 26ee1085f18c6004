set -x
mkdir -p gpurun_out/g15
timeout 900 python -m pytest tests/test_gpu_q4.py tests/test_gpu_prefill.py -q -x > gpurun_out/g15/q4.log 2>&1
B="python bench.py --no-cpu-baseline"
timeout 400 $B --config mixtral_prefill --steps 3 --e2e-steps 1 --weights q4 > gpurun_out/g15/prefill_q4.json 2> gpurun_out/g15/prefill_q4.err
timeout 400 $B --config mixtral_prefill --steps 3 --e2e-steps 1 > gpurun_out/g15/prefill_bf16.json 2> gpurun_out/g15/prefill_bf16.err
