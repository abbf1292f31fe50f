"""Split-K sweep for the long-K GEMMs of the step (weight gradients, OPM
da/dc): time each shape with EVO_GEMM_SPLITS forced to each candidate.

    python tools/splitk_sweep.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402

SHAPES = [  # M, N, K, ta, tb, out
    (256, 1024, 32768, 1, 0, "f32"), (1024, 128, 65536, 1, 0, "f32"), (1024, 256, 32768, 1, 0, "f32"),
    (128, 512, 65536, 1, 0, "f32"), (256, 256, 32768, 1, 0, "f32"), (128, 128, 65536, 1, 0, "f32"),
    (512, 128, 65536, 1, 0, "f32"), (128, 8192, 8192, 0, 1, "bf16"), (128, 8192, 8192, 0, 0, "bf16"),
    (256, 64, 32768, 1, 0, "f32"),
]


def t_us(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def main():
    for M, N, K, ta, tb, out in SHAPES:
        a = torch.randn((K, M) if ta else (M, K), device="cuda").bfloat16()
        b = torch.randn((N, K) if tb else (K, N), device="cuda").bfloat16()
        c = torch.empty((M, N), device="cuda", dtype=torch.bfloat16 if out == "bf16" else torch.float32)
        res = []
        for sp in (0, 1, 2, 4, 6, 8, 12, 16, 18, 24, 32, 48, 64):
            if sp:
                os.environ["EVO_GEMM_SPLITS"] = str(sp)
            else:
                os.environ.pop("EVO_GEMM_SPLITS", None)
            res.append((sp, t_us(lambda: ops.gemm(a, b, c, ta=bool(ta), tb=bool(tb)))))
        os.environ.pop("EVO_GEMM_SPLITS", None)
        best = min(res[1:], key=lambda r: r[1])
        print(f"M={M} N={N} K={K} ta={ta} tb={tb} {out}: default {res[0][1]:.1f} us, best splits={best[0]} "
              f"{best[1]:.1f} us | " + " ".join(f"{sp}:{u:.1f}" for sp, u in res[1:]), flush=True)


if __name__ == "__main__":
    main()
