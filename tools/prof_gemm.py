"""Run a few representative GEMMs once each (for ncu):

    ncu --set full -k regex:gemm_tc python tools/prof_gemm.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402

CASES = [  # M, N, K, ta, tb, out, epi
    (32768, 1024, 256, 0, 0, "bf16", "none"),     # qkvg projection
    (256, 1024, 32768, 1, 0, "f32", "none"),      # d[Wq|Wk|Wv|Wg]
    (128, 8192, 8192, 0, 1, "bf16", "none"),      # OPM da
    (32768, 256, 1024, 0, 1, "f32", "none"),      # dxl = dqkvg . wcat^T
    (32768, 256, 256, 0, 0, "bf16", "res"),       # output projection + bias + residual
]


def main():
    sel = [int(a) for a in sys.argv[1:]] or range(len(CASES))
    for i in sel:
        M, N, K, ta, tb, out, epi = CASES[i]
        a = torch.randn((K, M) if ta else (M, K), device="cuda").bfloat16()
        b = torch.randn((N, K) if tb else (K, N), device="cuda").bfloat16()
        c = torch.empty((M, N), device="cuda", dtype=torch.bfloat16 if out == "bf16" else torch.float32)
        for _ in range(2):
            if epi == "res":
                ops.gemm_bias(a, b, c, torch.zeros(N, device="cuda"), res=torch.zeros_like(c))
            else:
                ops.gemm(a, b, c, ta=bool(ta), tb=bool(tb))
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
