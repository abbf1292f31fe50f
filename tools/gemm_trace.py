"""Per-tile phase timeline of CTA 0 of one tcgen05 GEMM (a -DEVO_GEMM_TRACE
build, tools/build_trace.py gemm_tc):

    EVO_LIB_PATH=ab/trace/libevoformer_sm100.so python tools/gemm_trace.py M N K ta tb [f32]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import _lib, ops  # noqa: E402


def main(M=32768, N=1024, K=256, ta=0, tb=0, out="bf16"):
    M, N, K, ta, tb = int(M), int(N), int(K), int(ta), int(tb)
    a = torch.randn((K, M) if ta else (M, K), device="cuda").bfloat16()
    b = torch.randn((N, K) if tb else (K, N), device="cuda").bfloat16()
    c = torch.empty((M, N), device="cuda", dtype=torch.float32 if out == "f32" else torch.bfloat16)
    for _ in range(3):
        ops.gemm(a, b, c, ta=bool(ta), tb=bool(tb))
    torch.cuda.synchronize()
    buf = np.zeros(4096, dtype=np.int64)
    lib = _lib.lib()
    lib.evo_gemm_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.evo_gemm_trace_read(buf.ctypes.data, 4096)
    t0 = buf[511 * 8 + 7]
    print(f"M={M} N={N} K={K} ta={ta} tb={tb} {out}: cycles from CTA 0 start")
    print(" it  prod_start mma_wait_acc mma_has_acc mma_issued epi_tfull epi_done")
    for it in range(511):
        row = buf[it * 8:it * 8 + 8]
        if row[1] == 0 and row[5] == 0:
            break
        f = lambda v: f"{v - t0:10d}" if v else "         -"
        print(f"{it:3d} {f(row[5])} {f(row[0])} {f(row[1])} {f(row[2])} {f(row[3])} {f(row[4])}")


if __name__ == "__main__":
    main(*sys.argv[1:])
