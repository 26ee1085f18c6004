set -x
OUT=$PWD/gpurun_out/g36
mkdir -p $OUT
for r in 1 2; do
timeout 300 python scripts/k2_bench.py --cases mixtral:1,qwen3:1,deepseek:1 --steps 30 > $OUT/new_$r.jsonl 2> $OUT/new_$r.log
(cd _wt/old && timeout 300 python scripts/k2_bench.py --cases mixtral:1,qwen3:1,deepseek:1 --steps 30 > $OUT/old_$r.jsonl 2> $OUT/old_$r.log)
done
