"""CUDA-event timing of the attention core kernels at the bench shapes.

    python tools/time_attn.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    gr.replay()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    S, R, H = 128, 256, 8
    for which in ("tri", "row", "col"):
        C = 128 if which == "tri" else 256
        D = C // H
        if which == "tri":
            B, L, sb, sl, T, msb, msl = R, R, R, 1, R * R, R, 1
        elif which == "row":
            B, L, sb, sl, T, msb, msl = S, R, R, 1, S * R, R, 1
        else:
            B, L, sb, sl, T, msb, msl = R, S, 1, R, S * R, 1, R
        qkvg = (torch.randn(T, 4 * C, device="cuda") * 0.5).to(torch.bfloat16)
        mask = torch.ones(T, device="cuda")
        bias = (torch.randn(H, L, L, device="cuda") * 0.1).to(torch.bfloat16) if which != "col" else None
        bg = torch.zeros(C, device="cuda")
        ctx, gate, gated, lse = ops.attn_fwd(qkvg, mask, msb, msl, bias, bg, B, L, H, D, sb, sl)
        dg = torch.randn_like(ctx)
        dbg = torch.empty(C, device="cuda")
        tf = timeit(lambda: ops.attn_fwd(qkvg, mask, msb, msl, bias, bg, B, L, H, D, sb, sl))
        tb = timeit(lambda: ops.attn_bwd(qkvg, mask, msb, msl, bias, ctx, gate, dg, lse, dbg, B, L, H, D,
                                         sb, sl, want_dbias=bias is not None))
        if bias is not None and os.environ.get("ATTN_ABLATE"):
            tnb = timeit(lambda: ops.attn_bwd(qkvg, mask, msb, msl, bias, ctx, gate, dg, lse, dbg, B, L, H, D,
                                              sb, sl, want_dbias=False))
            tnn = timeit(lambda: ops.attn_bwd(qkvg, mask, msb, msl, None, ctx, gate, dg, lse, dbg, B, L, H, D,
                                              sb, sl, want_dbias=False))
            print(f"   ablation: bwd without d(bias) {tnb:8.1f} us, without bias at all {tnn:8.1f} us")
        exps = B * H * L * L
        print(f"{which}: B={B} L={L} H={H} D={D}  fwd {tf:8.1f} us  bwd(all kernels) {tb:8.1f} us  "
              f"ex2 bound {exps / (148 * 16 * 1.965e3):.1f} us")


if __name__ == "__main__":
    main()
