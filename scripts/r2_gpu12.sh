# reproducibility (3 headline runs), kernel-event overhead on the chain, router phases, 2-rank EP/TP lines
set -x
mkdir -p gpurun_out/g12
for r in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g12/mixtral_run$r.json 2> gpurun_out/g12/mixtral_run$r.err; done
B="python bench.py --no-cpu-baseline --e2e-steps 0"
for c in qwen3 deepseek; do
  timeout 300 $B --config $c --steps 32 --no-kernel-events > gpurun_out/g12/${c}_noev.json 2> gpurun_out/g12/${c}_noev.err
  timeout 300 $B --config $c --steps 32 --prefetch-window-us 80 --no-kernel-events > gpurun_out/g12/${c}_w80_noev.json 2> gpurun_out/g12/${c}_w80_noev.err
  MOEPIC_HOST_TIMING=1 MOEPIC_K1_TRACE=1 timeout 300 $B --config $c --steps 8 > gpurun_out/g12/${c}_trace.json 2> gpurun_out/g12/${c}_trace.err
done
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 2 --config deepseek --gpus 2 --dist-backend gloo --parallel ep --steps 8 > gpurun_out/g12/deepseek_ep2.json 2> gpurun_out/g12/deepseek_ep2.err
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 2 --config mixtral --gpus 2 --dist-backend gloo --parallel tp --steps 4 > gpurun_out/g12/mixtral_tp2.json 2> gpurun_out/g12/mixtral_tp2.err
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 --config mixtral_prefill --gpus 2 --dist-backend gloo --parallel ep --steps 3 > gpurun_out/g12/prefill_ep2.json 2> gpurun_out/g12/prefill_ep2.err
