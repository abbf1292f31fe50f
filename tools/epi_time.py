"""Graph-timed comparison of the fused transition epilogues (ReLU-aux fwd,
dReLU bwd, bias-grad-in-GEMM) against the unfused kernel sequences.

    python tools/epi_time.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402
from time_glue import timeit  # noqa: E402


def main():
    for T, C in ((65536, 128), (32768, 256)):
        F = 4 * C
        xl = torch.randn(T, C, device="cuda").bfloat16()
        w1 = (torch.randn(C, F, device="cuda") / C ** 0.5).bfloat16()
        w2 = (torch.randn(F, C, device="cuda") / F ** 0.5).bfloat16()
        b1 = torch.randn(F, device="cuda") * 0.1
        h = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
        ld = ops.relu_aux_ld(F)
        aux = torch.empty(T, ld // 8, dtype=torch.uint8, device="cuda")
        d_act = torch.randn(T, C, device="cuda").bfloat16()
        dh = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
        dw1 = torch.empty(C, F, device="cuda")
        db1 = torch.empty(F, device="cuda")
        t = {}
        t["fwd relu_aux_bias"] = timeit(lambda: ops.gemm_epilogue(xl, w1, h, 3, vec=b1, aux=aux, aux_ld=ld))
        t["fwd relu_bias   "] = timeit(lambda: ops.gemm_bias(xl, w1, h, b1, relu=True))
        t["bwd drelu        "] = timeit(lambda: ops.gemm_epilogue(d_act, w2, dh, 4, aux=aux, aux_ld=ld, tb=True))
        t["bwd gemm         "] = timeit(lambda: ops.gemm(d_act, w2, dh, tb=True))
        t["bwd relu_colsum  "] = timeit(lambda: ops.relu_bwd_colsum_(dh, h, db1))
        t["dW1 bgrada       "] = timeit(lambda: ops.gemm_epilogue(xl, dh, dw1, 5, vec=db1, ta=True))
        t["dW1 gemm         "] = timeit(lambda: ops.gemm(xl, dh, dw1, ta=True))
        for k, v in t.items():
            print(f"T={T} C={C}  {k} {v:8.1f} us")


if __name__ == "__main__":
    main()
