# round 2 re-entry: GPU suite + bench lines on every decode config, prefetch-window sweep
set -x
mkdir -p gpurun_out/g1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1/smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/g1/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g1/pytest_gpu.log 2>&1
B="python bench.py"
timeout 600 $B > gpurun_out/g1/mixtral.json 2> gpurun_out/g1/mixtral.err
B="python bench.py --no-cpu-baseline --e2e-steps 0"
for c in qwen3 deepseek; do
  timeout 300 $B --config $c --steps 32 > gpurun_out/g1/${c}.json 2> gpurun_out/g1/${c}.err
  for w in 40 80 160; do
    timeout 300 $B --config $c --steps 32 --prefetch-window-us $w > gpurun_out/g1/${c}_w$w.json 2> gpurun_out/g1/${c}_w$w.err
  done
done
timeout 300 $B --config mixtral_prefill --steps 3 > gpurun_out/g1/prefill.json 2> gpurun_out/g1/prefill.err
timeout 300 $B --config qwen3 --batch 16 --steps 16 > gpurun_out/g1/qwen3_b16.json 2> gpurun_out/g1/qwen3_b16.err
