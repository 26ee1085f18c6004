# ncu --set full of one gated K2 launch in the default bench after Alg. 1 (calibration tokens: the
# timed configuration; 705 MB algorithmic per launch at B = 1)
set -x
OUT=gpurun_out/g48
mkdir -p $OUT
for s in 6200 5200; do
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k2_split -s $s -c 1 -f -o $OUT/k2_gated_$s \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_$s.log 2>&1
python scripts/ncu_summary.py $OUT/k2_gated_$s.ncu-rep > $OUT/summary_k2_gated_$s.md 2>&1
ncu -i $OUT/k2_gated_$s.ncu-rep --page raw --csv > $OUT/k2_gated_${s}_raw.csv 2>&1
done
rm -f $OUT/*.ncu-rep
