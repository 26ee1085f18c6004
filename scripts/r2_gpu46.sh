# Round-2 final evidence pass (one GPU): GPU suite + smoke, the default bench line x3 (mean / sd),
# every config's line, Q4 / attention / reference arm, two ranks on the one GPU (gloo, EP and TP),
# the ncu launch list of the default bench and ncu --set full of a K2 launch inside the bench.
set -x
OUT=gpurun_out/g46
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_suite.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
for r in 1 2 3; do
  timeout 600 python bench.py > $OUT/bench_default_$r.json 2> $OUT/bench_default_$r.log
done
timeout 600 python bench.py --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_mixtral_32.json 2> $OUT/bench_mixtral_32.log
timeout 600 python bench.py --config qwen3 --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_qwen3.json 2> $OUT/bench_qwen3.log
timeout 600 python bench.py --config deepseek --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_deepseek.json 2> $OUT/bench_deepseek.log
timeout 600 python bench.py --config qwen3 --batch 16 --steps 16 --no-cpu-baseline > $OUT/bench_qwen3_b16.json 2> $OUT/bench_qwen3_b16.log
timeout 600 python bench.py --config toy --steps 32 > $OUT/bench_toy.json 2> $OUT/bench_toy.log
timeout 600 python bench.py --config mixtral_prefill --steps 4 --warmup 3 > $OUT/bench_prefill.json 2> $OUT/bench_prefill.log
timeout 600 python bench.py --config mixtral_prefill --steps 4 --warmup 3 --weights q4 --no-cpu-baseline > $OUT/bench_prefill_q4.json 2> $OUT/bench_prefill_q4.log
timeout 600 python bench.py --weights q4 --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_mixtral_q4.json 2> $OUT/bench_mixtral_q4.log
timeout 600 python bench.py --attention 4096 --steps 16 --warmup 3 --no-cpu-baseline > $OUT/bench_mixtral_attention.json 2> $OUT/bench_mixtral_attention.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.log
timeout 900 python bench.py --config deepseek --gpus 2 --dist-backend gloo --parallel ep --steps 8 --no-cpu-baseline --e2e-steps 2 > $OUT/bench_deepseek_ep2_gloo_1gpu.json 2> $OUT/bench_deepseek_ep2.log
timeout 900 python bench.py --config mixtral --gpus 2 --dist-backend gloo --parallel tp --steps 4 --no-cpu-baseline --e2e-steps 2 > $OUT/bench_mixtral_tp2_gloo_1gpu.json 2> $OUT/bench_mixtral_tp2.log
timeout 900 python bench.py --config mixtral_prefill --gpus 2 --dist-backend gloo --parallel ep --steps 3 --no-cpu-baseline --e2e-steps 1 > $OUT/bench_prefill_ep2_gloo_1gpu.json 2> $OUT/bench_prefill_ep2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/launches_bench.log 2>&1
python scripts/ncu_summary.py --launches $OUT/launches_bench.csv > $OUT/summary_launches.md 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_split_expert -s 3000 -c 1 -f -o $OUT/k2_bench_mixtral \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_k2_bench.log 2>&1
python scripts/ncu_summary.py $OUT/k2_bench_mixtral.ncu-rep > $OUT/summary_k2_bench_mixtral.md 2>&1
rm -f $OUT/*.ncu-rep $OUT/launches_bench.csv
