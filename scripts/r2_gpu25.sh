set -x
mkdir -p gpurun_out/g25
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 16"
for c in mixtral deepseek qwen3; do
  timeout 300 $B --config $c > gpurun_out/g25/${c}_moepic_auto.json 2> gpurun_out/g25/${c}_moepic_auto.err
  timeout 300 $B --config $c --prefetch-window-us 0 > gpurun_out/g25/${c}_moepic_w0.json 2> gpurun_out/g25/${c}_moepic_w0.err
done
