set -x
mkdir -p gpurun_out/e1
B="python bench.py --no-cpu-baseline"
$B --config toy --gpus 2 --dist-backend gloo --parallel tp --steps 4 > gpurun_out/e1/toy_tp2.json 2> gpurun_out/e1/toy_tp2.err
$B --config toy --gpus 2 --dist-backend gloo --parallel ep --steps 4 > gpurun_out/e1/toy_ep2.json 2> gpurun_out/e1/toy_ep2.err
$B --config mixtral_prefill --gpus 2 --dist-backend gloo --steps 2 --e2e-steps 1 > gpurun_out/e1/pf_ep2.json 2> gpurun_out/e1/pf_ep2.err
$B --config qwen3 --steps 32 > gpurun_out/e1/qwen3.json 2> gpurun_out/e1/qwen3.err
MOEPIC_NO_SOLVER_YCAP=1 $B --config qwen3 --steps 32 --y-cap 1 > gpurun_out/e1/qwen3_y1.json 2> gpurun_out/e1/qwen3_y1.err
$B --config deepseek --steps 32 > gpurun_out/e1/deepseek.json 2> gpurun_out/e1/deepseek.err
MOEPIC_NO_SOLVER_YCAP=1 $B --config deepseek --steps 32 --y-cap 1 > gpurun_out/e1/deepseek_y1.json 2> gpurun_out/e1/deepseek_y1.err
$B --config mixtral --steps 20 > gpurun_out/e1/mixtral.json 2> gpurun_out/e1/mixtral.err
