"""Attention fwd/bwd at a bench geometry: finiteness and agreement of the
bf16 tcgen05 path with the fp32 SIMT path on the same inputs.
    python tools/attn_check.py col|row|tri"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402


def main(which="col", S=128, R=256, H=8):
    S, R, H = int(S), int(R), int(H)
    C = 128 if which == "tri" else 256
    D = C // H
    if which == "tri":
        B, L, sb, sl, T, msb, msl = R, R, R, 1, R * R, R, 1
    elif which == "row":
        B, L, sb, sl, T, msb, msl = S, R, R, 1, S * R, R, 1
    else:
        B, L, sb, sl, T, msb, msl = R, S, 1, R, S * R, 1, R
    torch.manual_seed(0)
    q32 = torch.randn(T, 4 * C, device="cuda") * 0.5
    mask = torch.ones(T, device="cuda")
    nv = R - R // 10  # the bench features pad the last 10% of residues
    mv = mask.view(S, R) if which in ("row", "col") else mask.view(R, R)
    mv[:, nv:] = 0.0
    if which == "tri":
        mv[nv:, :] = 0.0
    bias32 = torch.randn(H, L, L, device="cuda") * 0.1 if which != "col" else None
    bg = torch.zeros(C, device="cuda")
    dg32 = torch.randn(T, C, device="cuda")
    res = {}
    for dt in (torch.float32, torch.bfloat16):
        q = q32.to(dt)
        bias = bias32.to(dt) if bias32 is not None else None
        ctx, gate, gated, lse = ops.attn_fwd(q, mask, msb, msl, bias, bg, B, L, H, D, sb, sl)
        dbg = torch.empty(C, device="cuda")
        dq, dnb = ops.attn_bwd(q, mask, msb, msl, bias, ctx, gate, dg32.to(dt), lse, dbg, B, L, H, D, sb, sl,
                               want_dbias=bias is not None)
        torch.cuda.synchronize()
        res[dt] = (ctx.float(), dq.float(), dnb)
        print(dt, "ctx finite", bool(torch.isfinite(ctx.float()).all()), "dq finite",
              bool(torch.isfinite(dq.float()).all()))
        bad = ~torch.isfinite(dq.float())
        if bad.any():
            rows = bad.any(1).nonzero().flatten()
            cols = bad.any(0).nonzero().flatten()
            print("  bad rows", rows.numel(), rows[:8].tolist(), "bad cols", cols.numel(), cols[:8].tolist())
    a, b = res[torch.float32], res[torch.bfloat16]
    for k, n in ((0, "ctx"), (1, "dqkvg")):
        d = (a[k] - b[k]).abs().max() / a[k].abs().max()
        print(n, "rel err bf16 vs fp32", float(d))


if __name__ == "__main__":
    main(*sys.argv[1:])
