set -x
mkdir -p gpurun_out/g20
ncu --set full --clock-control none --import-source on -k regex:pf_gemm -s 4 -c 4 -f -o gpurun_out/g20/pf python scripts/pf_bench.py --steps 3 > gpurun_out/g20/ncu_pf.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2t -s 3 -c 2 -f -o gpurun_out/g20/k2t_qwen python scripts/k2_bench.py --cases qwen3:16 --steps 6 > gpurun_out/g20/ncu_k2t.log 2>&1
python scripts/pf_bench.py --steps 10 > gpurun_out/g20/pf.txt 2>&1
python scripts/pf_bench.py --steps 10 --pair 1 > gpurun_out/g20/pf_pair1.txt 2>&1
python scripts/pf_bench.py --steps 10 --pair 0 > gpurun_out/g20/pf_pair0.txt 2>&1
