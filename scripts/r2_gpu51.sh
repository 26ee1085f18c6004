# prefill: resident + prefetched segments in one GEMM group (parity tests, bench A/B)
set -x
OUT=gpurun_out/g51
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_q4.py tests/test_gpu_ep.py tests/test_gpu_group.py -x -q > $OUT/gpu_tests.txt 2>&1
for r in 1 2; do
  timeout 600 python bench.py --config mixtral_prefill --steps 4 --warmup 3 --no-cpu-baseline > $OUT/bench_prefill_merge_$r.json 2> $OUT/bench_prefill_merge_$r.log
  MOEPIC_PF_MERGE_AB=0 timeout 600 python bench.py --config mixtral_prefill --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/bench_prefill_split_$r.json 2> $OUT/bench_prefill_split_$r.log
done
timeout 600 python bench.py --config mixtral_prefill --steps 4 --warmup 3 --weights q4 --no-cpu-baseline > $OUT/bench_prefill_q4.json 2> $OUT/bench_prefill_q4.log
