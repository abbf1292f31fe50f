"""Drive the OPM GEMM-epilogue kernels (evo_opm_outn / evo_opm_dnum) once each
at the bench shape, for an ncu capture of their DRAM bytes and warps active:

    ncu --set full --clock-control none -k regex:gemm_tc -o opm python tools/prof_opm.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402


def main():
    S, R, k, C = 128, 256, 32, 128
    a = torch.randn(S, R * k, device="cuda").bfloat16()
    c = torch.randn(S, R * k, device="cuda").bfloat16()
    rec = torch.rand(R * R, device="cuda")
    d_act = torch.randn(R * R, C, device="cuda").bfloat16()
    w_out = torch.randn(k * k, C, device="cuda").bfloat16()
    ops.opm_outn(a, c, rec, S, R, k)
    ops.opm_dnum(d_act, w_out, rec, R, k)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
