# K2 in-kernel time in the decode vs a resident layer: k2_bench with / without a saturated link,
# and per-CTA phase stamps of the decode's gated launches (MOEPIC_K2_TRACE syncs per launch)
set -x
OUT=gpurun_out/g34
mkdir -p $OUT
timeout 300 python scripts/k2_bench.py --cases mixtral:1,qwen3:1 --steps 30 > $OUT/k2_idle.jsonl 2> $OUT/k2_idle.log
timeout 300 python scripts/k2_bench.py --cases mixtral:1,qwen3:1 --steps 30 --pcie-load > $OUT/k2_load.jsonl 2> $OUT/k2_load.log
MOEPIC_K2_TRACE=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/trace_mixtral.json 2> $OUT/trace_mixtral.log
MOEPIC_K2_TRACE=1 MOEPIC_K2_GATE=0 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/trace_mixtral_nogate.json 2> $OUT/trace_mixtral_nogate.log
grep k2trace $OUT/trace_mixtral.log | tail -80 > $OUT/trace_mixtral_tail.txt
grep k2trace $OUT/trace_mixtral_nogate.log | tail -160 > $OUT/trace_mixtral_nogate_tail.txt
rm -f $OUT/trace_mixtral.log $OUT/trace_mixtral_nogate.log
