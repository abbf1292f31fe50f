"""Drive the attention kernels at the bench shapes (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402


def main(which="tri", reps=3, bwd=1):
    reps, bwd = int(reps), int(bwd)
    S, R, H = 128, 256, 8
    C = 128 if which == "tri" else 256
    D = C // H
    if which == "tri":
        B, L, sb, sl, T = R, R, R, 1, R * R
    elif which == "row":
        B, L, sb, sl, T = S, R, R, 1, S * R
    else:  # col
        B, L, sb, sl, T = R, S, 1, R, S * R
    qkvg = (torch.randn(T, 4 * C, device="cuda") * 0.5).to(torch.bfloat16)
    mask = torch.ones(T, device="cuda")
    bias = (torch.randn(H, L, L, device="cuda") * 0.1).to(torch.bfloat16) if which != "col" else None
    bg = torch.zeros(C, device="cuda")
    for _ in range(reps):
        ctx, gate, gated, lse = ops.attn_fwd(qkvg, mask, sb if which != "col" else 1,
                                             sl if which != "col" else R, bias, bg, B, L, H, D, sb, sl)
        if bwd:
            dg = torch.randn_like(ctx)
            dbg = torch.empty(C, device="cuda")
            ops.attn_bwd(qkvg, mask, sb if which != "col" else 1, sl if which != "col" else R, bias,
                         ctx, gate, dg, lse, dbg, B, L, H, D, sb, sl, want_dbias=bias is not None)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(*sys.argv[1:])
