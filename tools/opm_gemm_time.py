"""Timing of the OPM contractions at the bench shape in both orientations.

    python tools/opm_gemm_time.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402
from time_glue import timeit  # noqa: E402


def main():
    S, Rk = 128, 8192
    bf = torch.bfloat16
    a2 = torch.randn(S, Rk, device="cuda").to(bf)
    c2 = torch.randn(S, Rk, device="cuda").to(bf)
    dnum = torch.randn(Rk, Rk, device="cuda").to(bf)
    num = torch.empty(Rk, Rk, device="cuda", dtype=bf)
    da = torch.empty(S, Rk, device="cuda", dtype=bf)
    daT = torch.empty(Rk, S, device="cuda", dtype=bf)
    print("num = a^T c        ", timeit(lambda: ops.gemm(a2, c2, num, ta=True)))
    print("da = c dnum^T      ", timeit(lambda: ops.gemm(c2, dnum, da, tb=True)))
    print("dc = a dnum        ", timeit(lambda: ops.gemm(a2, dnum, da)))
    print("daT = dnum c^T     ", timeit(lambda: ops.gemm(dnum, c2, daT, tb=True)))
    print("dcT = dnum^T a^T   ", timeit(lambda: ops.gemm(dnum, a2, daT, ta=True, tb=True)))
    ac = torch.cat([c2, a2], 0)  # [2S, Rk]
    d2 = torch.empty(2 * S, Rk, device="cuda", dtype=bf)
    print("[da;x] = [c;a] dnum^T (M=256)", timeit(lambda: ops.gemm(ac, dnum, d2, tb=True)))


if __name__ == "__main__":
    main()
