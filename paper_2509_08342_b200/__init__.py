"""B200-native MoEpic split-expert MoE layer library (arXiv 2509.08342).

The product is libmoepic.so (include/moepic.h): CUDA kernels for sm_100a plus a C++ host
control plane.  This package holds its build script and a ctypes binding; importing
`paper_2509_08342_b200.api` fails loudly when the library has not been built.
"""
__all__ = ["build", "api"]
