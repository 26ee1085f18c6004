set -x
mkdir -p gpurun_out/g24
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 16"
for c in mixtral deepseek qwen3; do
  timeout 300 $B --config $c --prefetch-window-us 0 > gpurun_out/g24/${c}_moepic_w0.json 2> gpurun_out/g24/${c}_moepic_w0.err
  timeout 300 $B --config $c --alg1-inputs measured > gpurun_out/g24/${c}_moepic_meas.json 2> gpurun_out/g24/${c}_moepic_meas.err
  timeout 300 $B --config $c --alg1-inputs measured --prefetch-window-us 0 > gpurun_out/g24/${c}_moepic_meas_w0.json 2> gpurun_out/g24/${c}_moepic_meas_w0.err
  timeout 300 $B --config $c --mode lcp-prefetch > gpurun_out/g24/${c}_lcp_pf.json 2> gpurun_out/g24/${c}_lcp_pf.err
  timeout 300 $B --config $c --mode lru-prefetch --prefetch-window-us 0 > gpurun_out/g24/${c}_lru_w0.json 2> gpurun_out/g24/${c}_lru_w0.err
done
