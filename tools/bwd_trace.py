"""Phase timeline of attn_bwd_tc_kernel (CTA 0: softmax warps 0 and 15, the
MMA warp) from a -DEVO_BWD_TRACE build:

    python tools/build_trace.py attention_tc_bwd
    EVO_LIB_PATH=ab/trace/libevoformer_sm100.so python tools/bwd_trace.py [tri|row|col]

Per 64-key sub-chunk n (clock64 cycles from the first stamp):
  softmax: wS = waiting for S/dP, got = S/dP ready, arr = copied out + arrived,
           cmp = P/dS/bias math done, kv = previous chunk's dQ/dK/dV ready
           (sub-chunk 0 of a chunk), drn = drained, st = P/dS stored,
           pds = P/dS arrival (sub-chunk 1)
  mma:     wSf = waiting for the S/dP copy-out, sf = released, sdp = S/dP(n+1)
           issued, pds = P/dS ready (odd n), kv = dQ/dK/dV issued
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import _lib, ops  # noqa: E402


def main(which="tri", nshow=24):
    nshow = int(nshow)
    S, R, H = 128, 256, 8
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
    for _ in range(3):
        ops.attn_bwd(qkvg, mask, msb, msl, bias, ctx, gate, dg, lse, dbg, B, L, H, D, sb, sl,
                     want_dbias=bias is not None)
    torch.cuda.synchronize()
    buf = np.zeros(8192, dtype=np.int64)
    lib = _lib.lib()
    lib.evo_bwd_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.evo_bwd_trace_read(buf.ctypes.data, 8192)
    t0 = buf[buf > 0].min()
    rel = lambda v: v - t0 if v > 0 else -1  # noqa: E731
    sn = ["wS", "got", "arr", "cmp", "kv", "drn", "st", "pds"]
    mn = ["wSf", "sf", "sdp", "pds", "kv"]
    n = 0
    while n < 128 and buf[16 * n + 1] > 0:
        n += 1
    span = []
    for i in range(n):
        for base, tag in ((0, "w0 "), (4096, "w15")):
            ev = [rel(v) for v in buf[base + 16 * i: base + 16 * i + 8]]
            if i < nshow:
                print(f"n={i:3d} {tag} " + " ".join(f"{a}={b:7d}" for a, b in zip(sn, ev)))
        mm = [rel(v) for v in buf[2048 + 8 * i: 2048 + 8 * i + 5]]
        if i < nshow:
            print(f"n={i:3d} mma " + " ".join(f"{a}={b:7d}" for a, b in zip(mn, mm)))
        if i > 0:
            span.append(buf[16 * i + 1] - buf[16 * (i - 1) + 1])
    sp = np.array(span[4:])
    print(f"{n} sub-chunks; cycles per sub-chunk (S ready to S ready, warp 0): median {np.median(sp):.0f} "
          f"mean {sp.mean():.0f}")
    # mean phase durations (warp 0)
    w = buf[:16 * n].reshape(n, 16)[:, :8].astype(np.float64)
    for a, b, nm in ((0, 1, "wait S/dP"), (1, 2, "copy-out+arrive"), (2, 3, "P/dS math"), (3, 6, "kv wait+drain+store")):
        d = w[4:, b] - w[4:, a]
        print(f"  warp0 {nm:22s} mean {d.mean():7.0f} cycles")


if __name__ == "__main__":
    main(*sys.argv[1:])
