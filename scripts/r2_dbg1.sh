mkdir -p gpurun_out/d1
MOEPIC_POISON=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "od_tail_split" > gpurun_out/d1/a_cs2.log 2>&1
MOEPIC_COPY_STREAMS=1 MOEPIC_POISON=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "od_tail_split" > gpurun_out/d1/b_cs1.log 2>&1
MOEPIC_K2T=0 MOEPIC_POISON=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "od_tail_split" > gpurun_out/d1/c_nok2t.log 2>&1
MOEPIC_OD_SPLIT_BOUNDARY=0 MOEPIC_POISON=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "od_tail_split" > gpurun_out/d1/d_nobound.log 2>&1
MOEPIC_POISON=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_k2t.py -q > gpurun_out/d1/e_all.log 2>&1
