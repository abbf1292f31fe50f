"""Phase timeline of attn_fwd_tc2 (CTA 0) from a -DEVO_F2_TRACE build:

    EVO_LIB_PATH=build/trace/libevoformer_sm100.so python tools/f2_trace.py [tri|row|col]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import _lib, ops  # noqa: E402


def main(which="tri"):
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
    for _ in range(3):
        ops.attn_fwd(qkvg, mask, msb, msl, bias, bg, B, L, H, D, sb, sl)
    torch.cuda.synchronize()
    buf = np.zeros(8192, dtype=np.int64)
    lib = _lib.lib()
    lib.evo_f2_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.evo_f2_trace_read(buf.ctypes.data, 8192)
    t0 = buf[buf > 0].min()
    names = ["wait_s", "s_ready", "pass1", "pass2", "wait_o", "o_ready", "done"]
    nb = 0
    while buf[16 * nb + 1] > 0:
        nb += 1
    for n in range(nb):
        ev = buf[16 * n:16 * n + 7] - t0
        mm = buf[2048 + 8 * n:2048 + 8 * n + 4] - t0
        print(f"n={n:3d} wg{n % 2} " + " ".join(f"{nm}={v:7d}" for nm, v in zip(names, ev)) +
              f" | mma: wait_p={mm[0]:7d} p_ok={mm[1]:7d} tfree_ok={mm[2]:7d} s_issued={mm[3]:7d}")


if __name__ == "__main__":
    main(*sys.argv[1:])
