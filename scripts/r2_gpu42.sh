set -x
OUT=gpurun_out/g42
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_tp.py tests/test_gpu_ep.py tests/test_gpu_group.py -q > $OUT/gpu_tests.txt 2>&1
