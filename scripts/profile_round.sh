#!/bin/bash
# One GPU pass that regenerates the round's evidence under gpurun_out/ (summarised into profiles/
# by scripts/ncu_summary.py / ncu_traffic.py): bench lines for every config, the reference arm,
# the ncu launch list of the default bench, ncu --set full captures of K2 (resident layers and
# in the decode step) and of the router.  Never time anything under ncu.
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
python bench.py --steps 32 --warmup 3 > $OUT/bench_mixtral.json 2> $OUT/bench_mixtral.log
for c in qwen3 deepseek toy; do
  python bench.py --config $c --steps 32 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.log
done
python bench.py --config mixtral_prefill --steps 4 --warmup 3 > $OUT/bench_mixtral_prefill.json 2> $OUT/bench_mixtral_prefill.log
python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference_mixtral.json 2> $OUT/bench_reference.log
python bench.py --weights q4 --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_mixtral_q4.json 2> $OUT/bench_mixtral_q4.log
python bench.py --attention 4096 --steps 16 --warmup 3 --no-cpu-baseline > $OUT/bench_mixtral_attention.json 2> $OUT/bench_mixtral_attention.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/launches_bench.log 2>&1
for c in mixtral qwen3 deepseek; do
  ncu --set full --clock-control none --import-source on -k regex:k2_split_expert -s 5 -c 2 -f -o $OUT/k2_$c \
      python scripts/k2_bench.py --cases $c:1 --steps 3 > $OUT/ncu_k2_$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k1_router -s 5 -c 2 -f -o $OUT/k1_qwen3 \
    python scripts/k2_bench.py --cases qwen3:1 --steps 3 > $OUT/ncu_k1_qwen3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_attn -s 64 -c 2 -f -o $OUT/attn_mixtral \
    python bench.py --attention 4096 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-adapt > $OUT/ncu_attn.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_split_expert -s 300 -c 3 -f -o $OUT/k2_step_mixtral \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-adapt > $OUT/ncu_k2_step.log 2>&1
# summaries on the box; the reports themselves stay there (gpurun copies back <= 64 MiB)
python scripts/ncu_summary.py --launches $OUT/launches_bench.csv > $OUT/summary_launches.md 2>&1
for r in k2_mixtral k2_qwen3 k2_deepseek k2_step_mixtral k1_qwen3 attn_mixtral; do
  python scripts/ncu_summary.py $OUT/$r.ncu-rep > $OUT/summary_$r.md 2>&1
done
python scripts/ncu_traffic.py --out $OUT/ncu_traffic.json --k2 mixtral=$OUT/k2_mixtral.ncu-rep qwen3=$OUT/k2_qwen3.ncu-rep \
    deepseek=$OUT/k2_deepseek.ncu-rep --k2-bytes mixtral=704660000 qwen3=75530000 deepseek=138440000 > /dev/null 2>&1
rm -f $OUT/*.ncu-rep $OUT/launches_bench.csv
ls -la $OUT
