# same-box A/B of K2 on resident layers: current tree vs HEAD~ (14de0fe) vs the fp16-down commit
set -x
OUT=$PWD/gpurun_out/g35
mkdir -p $OUT
for r in 1 2; do
timeout 300 python scripts/k2_bench.py --cases mixtral:1,qwen3:1 --steps 30 > $OUT/new_$r.jsonl 2> $OUT/new_$r.log
MOEPIC_PDL=0 timeout 300 python scripts/k2_bench.py --cases mixtral:1,qwen3:1 --steps 30 > $OUT/new_nopdl_$r.jsonl 2> $OUT/new_nopdl_$r.log
(cd _wt/old && timeout 300 python scripts/k2_bench.py --cases mixtral:1,qwen3:1 --steps 30 > $OUT/old_$r.jsonl 2> $OUT/old_$r.log)
(cd _wt/fp16 && timeout 300 python scripts/k2_bench.py --cases mixtral:1,qwen3:1 --steps 30 > $OUT/fp16_$r.jsonl 2> $OUT/fp16_$r.log)
done
