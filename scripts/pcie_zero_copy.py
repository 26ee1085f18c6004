"""Probe (tools only): SM loads from mapped pinned memory vs the copy engine over PCIe, alone and
concurrently (scripts/pcie_zero_copy.cu).  Prints one JSON line per launch shape."""
import ctypes
import json
import os

so = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_zc.so"))
out = (ctypes.c_double * 5)()
for blocks, threads in ((148, 512), (296, 512), (592, 1024), (1184, 1024)):
    rc = so.zc_probe(ctypes.c_size_t(1 << 30), blocks, threads, out)
    print(json.dumps({"blocks": blocks, "threads": threads, "rc": rc,
                      "zc_alone_gbs": round(out[0], 2), "dma_alone_gbs": round(out[1], 2),
                      "zc_with_dma_gbs": round(out[2], 2), "dma_with_zc_gbs": round(out[3], 2),
                      "combined_gbs": round(out[4], 2)}))
