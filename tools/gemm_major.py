"""Time one GEMM shape with every operand-major combination (is an
MN-major operand slower on the tensor core?).

    python tools/gemm_major.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for (M, N, K) in [(256, 1024, 32768), (1024, 1024, 8192), (8192, 1024, 1024), (32768, 256, 1024)]:
    for ta in (0, 1):
        for tb in (0, 1):
            a = torch.randn((K, M) if ta else (M, K), device="cuda").bfloat16()
            b = torch.randn((N, K) if tb else (K, N), device="cuda").bfloat16()
            c = torch.empty((M, N), device="cuda", dtype=torch.float32)
            us = timeit(lambda: ops.gemm(a, b, c, ta=bool(ta), tb=bool(tb)))
            print(f"M={M:6d} N={N:5d} K={K:6d} A{'mn' if ta else 'k '} B{'k ' if tb else 'mn'} {us:7.1f} us "
                  f"{2 * M * N * K / us / 1e6:7.1f} TF/s")
