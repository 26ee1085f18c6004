set -x
mkdir -p gpurun_out/g21
B="python bench.py --no-cpu-baseline --e2e-steps 0"
for r in 1 2; do
for c in qwen3 deepseek; do
  timeout 300 $B --config $c --steps 32 > gpurun_out/g21/${c}_auto_$r.json 2> gpurun_out/g21/${c}_auto_$r.err
  timeout 300 $B --config $c --steps 32 --prefetch-window-us 0 > gpurun_out/g21/${c}_w0_$r.json 2> gpurun_out/g21/${c}_w0_$r.err
  timeout 300 $B --config $c --steps 32 --prefetch-window-us 30 > gpurun_out/g21/${c}_w30_$r.json 2> gpurun_out/g21/${c}_w30_$r.err
done
done
