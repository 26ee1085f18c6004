set -x
mkdir -p gpurun_out/g4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2t -s 3 -c 2 -o gpurun_out/g4/k2t_qwen python scripts/k2_bench.py --cases qwen3:16 --steps 6 > gpurun_out/g4/ncu_q.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2t -s 3 -c 2 -o gpurun_out/g4/k2t_ds python scripts/k2_bench.py --cases deepseek:16 --steps 6 > gpurun_out/g4/ncu_d.log 2>&1
