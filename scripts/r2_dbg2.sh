mkdir -p gpurun_out/d2
T="tests/test_gpu_parity.py::test_deepseek_shape_shared_no_renorm tests/test_gpu_k2t.py tests/test_gpu_parity.py::test_od_tail_split"
for r in 1 2; do
MOEPIC_POISON=1 MOEPIC_PDL=0 timeout 300 python -m pytest $T -q > gpurun_out/d2/nopdl_$r.log 2>&1
MOEPIC_POISON=1 MOEPIC_OD_SPLIT_BOUNDARY=0 timeout 300 python -m pytest $T -q > gpurun_out/d2/nobound_$r.log 2>&1
MOEPIC_POISON=1 timeout 300 python -m pytest $T -q > gpurun_out/d2/all_$r.log 2>&1
done
