# Round-2 evidence pass after the gated K2 (one launch per decode layer): GPU suite, smoke, the
# default bench line three times (mean / sd), Qwen3 / DeepSeek / B=16 / prefill lines, the ncu
# launch list of the default bench and one ncu --set full capture of a K2 launch inside the bench.
set -x
OUT=gpurun_out/g33
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_suite.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
for r in 1 2 3; do
  timeout 600 python bench.py > $OUT/bench_default_$r.json 2> $OUT/bench_default_$r.log
done
timeout 600 python bench.py --config qwen3 --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_qwen3.json 2> $OUT/bench_qwen3.log
timeout 600 python bench.py --config deepseek --steps 32 --warmup 3 --no-cpu-baseline > $OUT/bench_deepseek.json 2> $OUT/bench_deepseek.log
timeout 600 python bench.py --config qwen3 --batch 16 --steps 16 --no-cpu-baseline > $OUT/bench_qwen3_b16.json 2> $OUT/bench_qwen3_b16.log
timeout 600 python bench.py --config mixtral_prefill --steps 4 --warmup 3 --no-cpu-baseline > $OUT/bench_prefill.json 2> $OUT/bench_prefill.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/launches_bench.log 2>&1
python scripts/ncu_summary.py --launches $OUT/launches_bench.csv > $OUT/summary_launches.md 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_split_expert -s 3000 -c 1 -f -o $OUT/k2_bench_mixtral \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_k2_bench.log 2>&1
python scripts/ncu_summary.py $OUT/k2_bench_mixtral.ncu-rep > $OUT/summary_k2_bench_mixtral.md 2>&1
ncu -i $OUT/k2_bench_mixtral.ncu-rep --page raw --csv > $OUT/k2_bench_mixtral_raw.csv 2>&1
rm -f $OUT/*.ncu-rep $OUT/launches_bench.csv
