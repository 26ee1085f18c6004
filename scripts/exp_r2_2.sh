mkdir -p gpurun_out/e2
B="python bench.py --no-cpu-baseline --e2e-steps 0"
$B --config qwen3 --steps 32 --no-kernel-events > gpurun_out/e2/qwen3_noev.json 2> gpurun_out/e2/qwen3_noev.err
MOEPIC_NO_SOLVER_YCAP=1 $B --config qwen3 --steps 32 --y-cap 1 --no-kernel-events > gpurun_out/e2/qwen3_y1_noev.json 2> gpurun_out/e2/qwen3_y1_noev.err
$B --config deepseek --steps 32 --no-kernel-events > gpurun_out/e2/deepseek_noev.json 2> gpurun_out/e2/deepseek_noev.err
MOEPIC_NO_SOLVER_YCAP=1 $B --config deepseek --steps 32 --y-cap 1 --no-kernel-events > gpurun_out/e2/deepseek_y1_noev.json 2> gpurun_out/e2/deepseek_y1_noev.err
MOEPIC_HOST_TIMING=1 $B --config qwen3 --steps 32 --no-kernel-events > gpurun_out/e2/qwen3_ht.json 2> gpurun_out/e2/qwen3_ht.err
$B --config mixtral --steps 20 --no-kernel-events > gpurun_out/e2/mixtral_noev.json 2> gpurun_out/e2/mixtral_noev.err
