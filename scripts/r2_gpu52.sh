# final HEAD check: GPU suite, smoke, default bench line
set -x
OUT=gpurun_out/g52
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_suite.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.log
