"""Attention fwd/bwd timing at the fine-tune shape F (N_seq=512, N_res=384)
and the stress shape X (N_res=1024 triangle attention, forward only).
    python tools/time_attn_large.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402
from time_glue import timeit  # noqa: E402


def case(name, B, L, H, D, sb, sl, T, msb, msl, bias, bwd=True, reps=3):
    qkvg = (torch.randn(T, 4 * H * D, device="cuda") * 0.5).to(torch.bfloat16)
    mask = torch.ones(T, device="cuda")
    nb = (torch.randn(H, L, L, device="cuda") * 0.1).to(torch.bfloat16) if bias else None
    bg = torch.zeros(H * D, device="cuda")
    tf = timeit(lambda: ops.attn_fwd(qkvg, mask, msb, msl, nb, bg, B, L, H, D, sb, sl), reps=reps)
    tb = float("nan")
    if bwd:
        ctx, gate, gated, lse = ops.attn_fwd(qkvg, mask, msb, msl, nb, bg, B, L, H, D, sb, sl)
        dg = torch.randn_like(ctx)
        dbg = torch.empty(H * D, device="cuda")
        tb = timeit(lambda: ops.attn_bwd(qkvg, mask, msb, msl, nb, ctx, gate, dg, lse, dbg, B, L, H, D, sb, sl,
                                         want_dbias=bias), reps=reps)
    print(f"{name}: B={B} L={L} H={H} D={D}  fwd {tf:9.1f} us  bwd {tb:9.1f} us  "
          f"ex2 bound {B * H * L * L / (148 * 16 * 1.965e3):.1f} us")


def main():
    S, R, H = 512, 384, 8
    case("F row", S, R, H, 32, R, 1, S * R, R, 1, True)
    case("F col", R, S, H, 32, 1, R, S * R, 1, R, False)
    case("F tri", R, R, H, 16, R, 1, R * R, R, 1, True)
    X = 1024
    case("X tri (fwd)", X, X, 4, 32, X, 1, X * X, X, 1, True, bwd=False, reps=1)


if __name__ == "__main__":
    main()
