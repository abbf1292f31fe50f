"""Graph-replay timing of the triangle attention's input LayerNorm + pair bias:
two ops (layernorm, pair_bias_fwd) against the fused one-pass kernel.

    python tools/time_ln_pb.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402
from time_attn import timeit  # noqa: E402


def main():
    R, C, H = 256, 128, 8
    z = torch.randn(R * R, C, device="cuda").bfloat16()
    lg, lb, g, b = (torch.randn(C, device="cuda") for _ in range(4))
    w = torch.randn(C, H, device="cuda") * 0.2
    for swap in (0, 1):
        t2 = timeit(lambda: (ops.layernorm(z, lg, lb, torch.bfloat16), ops.pair_bias_fwd(z, g, b, w, R, H, swap)))
        t1 = timeit(lambda: ops.ln_pair_bias_fwd(z, lg, lb, g, b, w, R, H, swap))
        print(f"swap={swap}: layernorm + pair_bias_fwd {t2:6.1f} us, fused {t1:6.1f} us")


if __name__ == "__main__":
    main()
