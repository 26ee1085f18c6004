# auto prefetch window (measured link idle -> Alg. 1 T_att + plan cut), dominant-kernel-only events
set -x
mkdir -p gpurun_out/g14

B="python bench.py --no-cpu-baseline --e2e-steps 0"
for c in qwen3 deepseek; do
  timeout 300 $B --config $c --steps 32 > gpurun_out/g14/${c}_auto.json 2> gpurun_out/g14/${c}_auto.err
  timeout 300 $B --config $c --steps 32 --prefetch-window-us 0 > gpurun_out/g14/${c}_w0.json 2> gpurun_out/g14/${c}_w0.err
done
timeout 300 $B --config mixtral --steps 20 > gpurun_out/g14/mixtral_auto.json 2> gpurun_out/g14/mixtral_auto.err
timeout 300 $B --config mixtral --steps 20 --prefetch-window-us 0 > gpurun_out/g14/mixtral_w0.json 2> gpurun_out/g14/mixtral_w0.err
timeout 300 $B --config qwen3 --batch 16 --steps 16 > gpurun_out/g14/qwen3_b16_auto.json 2> gpurun_out/g14/qwen3_b16_auto.err
