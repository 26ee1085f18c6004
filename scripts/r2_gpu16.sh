# boundary split of the last on-demand copy + PDL router: A/B on the decode configs
set -x
mkdir -p gpurun_out/g16
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g16/pytest_gpu.log 2>&1
B="python bench.py --no-cpu-baseline --e2e-steps 0 --prefetch-window-us 0"
for c in qwen3 deepseek; do
  timeout 300 $B --config $c --steps 32 > gpurun_out/g16/${c}_new.json 2> gpurun_out/g16/${c}_new.err
  MOEPIC_PDL=0 timeout 300 $B --config $c --steps 32 > gpurun_out/g16/${c}_nopdl.json 2> gpurun_out/g16/${c}_nopdl.err
  MOEPIC_OD_SPLIT_BOUNDARY=0 MOEPIC_PDL=0 timeout 300 $B --config $c --steps 32 > gpurun_out/g16/${c}_old.json 2> gpurun_out/g16/${c}_old.err
done
timeout 300 $B --config mixtral --steps 16 > gpurun_out/g16/mixtral_new.json 2> gpurun_out/g16/mixtral_new.err
MOEPIC_PDL=0 timeout 300 $B --config mixtral --steps 16 > gpurun_out/g16/mixtral_nopdl.json 2> gpurun_out/g16/mixtral_nopdl.err
