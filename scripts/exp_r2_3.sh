mkdir -p gpurun_out/e3
B="python bench.py --no-cpu-baseline --e2e-steps 0"
for c in qwen3 deepseek; do
  $B --config $c --steps 32 > gpurun_out/e3/${c}_ev.json 2> gpurun_out/e3/${c}_ev.err
  $B --config $c --steps 32 --no-kernel-events > gpurun_out/e3/${c}_noev.json 2> gpurun_out/e3/${c}_noev.err
  for w in 30 60 90 150; do
    $B --config $c --steps 32 --no-kernel-events --prefetch-window-us $w > gpurun_out/e3/${c}_w$w.json 2> gpurun_out/e3/${c}_w$w.err
  done
done
$B --config mixtral --steps 16 > gpurun_out/e3/mixtral_ev.json 2> gpurun_out/e3/mixtral_ev.err
$B --config mixtral --steps 16 --no-kernel-events > gpurun_out/e3/mixtral_noev.json 2> gpurun_out/e3/mixtral_noev.err
$B --config mixtral --steps 16 --no-kernel-events --prefetch-window-us 60 > gpurun_out/e3/mixtral_w60.json 2> gpurun_out/e3/mixtral_w60.err
$B --config mixtral --steps 16 --no-kernel-events --prefetch-window-us 150 > gpurun_out/e3/mixtral_w150.json 2> gpurun_out/e3/mixtral_w150.err
