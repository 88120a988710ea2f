"""Random-row gather ceiling on this GPU (context for the aggregation kernels' roofline): a
warp sums U random rows of an [N x F] fp32 table per output row (indices precomputed, so
only memory-level parallelism limits it).  Build: nvcc -shared of tools/gather_bench.cu."""
import ctypes
import os
import subprocess

import torch

here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "libgather_bench.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode",
                           "arch=compute_100a,code=sm_100a", "-o", so, os.path.join(here, "gather_bench.cu")])
lib = ctypes.CDLL(so)
lib.gather_bench.restype = ctypes.c_float
N = 2_449_029
for F in (100, 256):
    X = torch.randn(N, F, device="cuda")
    for R in (532_000, 4_000_000):
        idx = torch.randint(0, N, (R,), device="cuda", dtype=torch.int32)
        for U in (1, 2, 4, 8, 16):
            out = torch.empty((R + U - 1) // U, F, device="cuda")
            for blocks in (148 * 8, 148 * 32):
                us = lib.gather_bench(ctypes.c_void_p(X.data_ptr()), F, ctypes.c_void_p(idx.data_ptr()), R,
                                      ctypes.c_void_p(out.data_ptr()), U, blocks, 10)
                rd = R * F * 4
                print(f"F={F} R={R} U={U:2d} blocks={blocks}: {us:7.1f} us  read {rd/us/1e3:6.0f} GB/s")
