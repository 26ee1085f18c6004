#!/bin/bash
# Round-2 evidence pass (one GPU): bench lines for every config, the reference arm, two-rank
# (gloo, one GPU) EP / TP lines, the ncu launch list of the default bench and ncu --set full
# captures of the dominant kernels (K2, K2T, prefill GEMMs, router).  Summaries are written next
# to the reports; the reports stay on the box.  Never time anything under ncu.
OUT=${OUT:-gpurun_out/p2}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
python bench.py --steps 32 --warmup 3 > $OUT/bench_mixtral.json 2> $OUT/bench_mixtral.log
for c in qwen3 deepseek; do
  python bench.py --config $c --steps 32 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.log
done
python bench.py --config qwen3 --batch 16 --steps 16 --no-cpu-baseline > $OUT/bench_qwen3_b16.json 2> $OUT/bench_qwen3_b16.log
python bench.py --config toy --steps 32 > $OUT/bench_toy.json 2> $OUT/bench_toy.log
python bench.py --config mixtral_prefill --steps 4 --warmup 3 > $OUT/bench_mixtral_prefill.json 2> $OUT/bench_mixtral_prefill.log
python bench.py --config mixtral_prefill --steps 4 --warmup 3 --weights q4 --no-cpu-baseline > $OUT/bench_mixtral_prefill_q4.json 2> $OUT/bench_mixtral_prefill_q4.log
python bench.py --weights q4 --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_mixtral_q4.json 2> $OUT/bench_mixtral_q4.log
python bench.py --attention 4096 --steps 16 --warmup 3 --no-cpu-baseline > $OUT/bench_mixtral_attention.json 2> $OUT/bench_mixtral_attention.log
python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference_mixtral.json 2> $OUT/bench_reference.log
python bench.py --config deepseek --gpus 2 --dist-backend gloo --parallel ep --steps 8 --no-cpu-baseline --e2e-steps 2 > $OUT/bench_deepseek_ep2_gloo_1gpu.json 2> $OUT/bench_deepseek_ep2.log
python bench.py --config mixtral --gpus 2 --dist-backend gloo --parallel tp --steps 4 --no-cpu-baseline --e2e-steps 2 > $OUT/bench_mixtral_tp2_gloo_1gpu.json 2> $OUT/bench_mixtral_tp2.log
python bench.py --config mixtral_prefill --gpus 2 --dist-backend gloo --parallel ep --steps 3 --no-cpu-baseline --e2e-steps 1 > $OUT/bench_prefill_ep2_gloo_1gpu.json 2> $OUT/bench_prefill_ep2.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/launches_bench.log 2>&1
for c in mixtral qwen3 deepseek; do
  ncu --set full --clock-control none --import-source on -k regex:k2_split_expert -s 5 -c 2 -f -o $OUT/k2_$c \
      python scripts/k2_bench.py --cases $c:1 --steps 3 > $OUT/ncu_k2_$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k2t -s 3 -c 2 -f -o $OUT/k2t_qwen3_b16 \
    python scripts/k2_bench.py --cases qwen3:16 --steps 6 > $OUT/ncu_k2t.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pf_gemm -s 4 -c 4 -f -o $OUT/pf_mixtral \
    python scripts/pf_bench.py --steps 3 > $OUT/ncu_pf.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_router -s 5 -c 2 -f -o $OUT/k1_qwen3 \
    python scripts/k2_bench.py --cases qwen3:1 --steps 3 > $OUT/ncu_k1_qwen3.log 2>&1
python scripts/ncu_summary.py --launches $OUT/launches_bench.csv > $OUT/summary_launches.md 2>&1
for r in k2_mixtral k2_qwen3 k2_deepseek k2t_qwen3_b16 pf_mixtral k1_qwen3; do
  python scripts/ncu_summary.py $OUT/$r.ncu-rep > $OUT/summary_$r.md 2>&1
done
cp profiles/ncu_traffic.json $OUT/ncu_traffic.json
python scripts/ncu_traffic.py --out $OUT/ncu_traffic.json --k2 mixtral=$OUT/k2_mixtral.ncu-rep qwen3=$OUT/k2_qwen3.ncu-rep \
    deepseek=$OUT/k2_deepseek.ncu-rep --k2-bytes mixtral=704660000 qwen3=75530000 deepseek=138440000 > /dev/null 2>&1
rm -f $OUT/*.ncu-rep $OUT/launches_bench.csv
ls -la $OUT
