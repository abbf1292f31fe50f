"""OPM backward d(pair) -> d(num): fused tcgen05 kernel vs GEMM + re-layout.

    python tools/opm_dnum_time.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402
from time_glue import timeit  # noqa: E402


def main():
    R, k, C = 256, 32, 128
    d_act = torch.randn(R * R, C, device="cuda").bfloat16()
    w_out = torch.randn(k * k, C, device="cuda").bfloat16()
    rec = torch.rand(R * R, device="cuda")
    doutn = torch.empty(R * R, k * k, device="cuda", dtype=torch.bfloat16)
    print("fused opm_dnum        ", timeit(lambda: ops.opm_dnum(d_act, w_out, rec, R, k)))
    print("gemm doutn            ", timeit(lambda: ops.gemm(d_act, w_out, doutn, tb=True)))
    print("opm_norm_bwd relayout ", timeit(lambda: ops.opm_norm_bwd(doutn, rec, R, k, torch.bfloat16)))


if __name__ == "__main__":
    main()


def outn():
    S, R, k = 128, 256, 32
    a = torch.randn(S, R * k, device="cuda").bfloat16()
    c = torch.randn(S, R * k, device="cuda").bfloat16()
    rec = torch.rand(R * R, device="cuda")
    print("fused opm_outn        ", timeit(lambda: ops.opm_outn(a, c, rec, S, R, k)))


if __name__ == "__main__":
    outn()
