"""CUDA-event timing of the bandwidth-bound glue kernels at the bench shapes,
reported against their algorithmic bytes.

    python tools/time_glue.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402

BF, F32 = torch.bfloat16, torch.float32


def timeit(fn, reps=30):
    """Device time per call: the calls are captured into a CUDA graph and
    replayed, so host (ctypes) overhead does not floor the measurement."""
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


def report(name, us, nbytes):
    print(f"{name:34s} {us:8.1f} us  {nbytes / 1e6:8.1f} MB  {nbytes / us / 1e3:7.0f} GB/s")


def main():
    dev = "cuda"
    R, S, cz, cm, H = 256, 128, 128, 256, 8
    for rows, C, tag in ((R * R, cz, "pair"), (S * R, cm, "msa")):
        x = torch.randn(rows, C, device=dev).to(BF)
        g, b = torch.ones(C, device=dev), torch.zeros(C, device=dev)
        us = timeit(lambda: ops.layernorm(x, g, b, BF))
        report(f"ln_fwd[{tag}] bf16->bf16", us, rows * C * 4 + rows * 8)
        y, mean, rstd = ops.layernorm(x, g, b, BF)
        dy = torch.randn(rows, C, device=dev)
        dres = torch.randn(rows, C, device=dev)
        dx = torch.empty(rows, C, device=dev)
        dg, db = torch.empty(C, device=dev), torch.empty(C, device=dev)
        us = timeit(lambda: ops.layernorm_bwd(x, dy, mean, rstd, g, dres, dx, dg, db))
        report(f"ln_bwd[{tag}] x16 dy32 dres32 dx32", us, rows * C * (2 + 4 + 4 + 4) + rows * 8)
        res = torch.randn(rows, C, device=dev).to(BF)
        yy = torch.randn(rows, C, device=dev).to(BF)
        out = torch.empty(rows, C, device=dev, dtype=BF)
        us = timeit(lambda: ops.bias_residual(res, yy, g, out))
        report(f"bias_residual[{tag}] bf16", us, rows * C * 6)
        h = torch.randn(rows, 4 * C, device=dev).to(BF)
        us = timeit(lambda: ops.bias_relu_(h, torch.zeros(4 * C, device=dev)))
        report(f"bias_relu[{tag}] bf16 x{4 * C}", us, rows * 4 * C * 4)
        dh = torch.randn(rows, 4 * C, device=dev).to(BF)
        db4 = torch.empty(4 * C, device=dev)
        us = timeit(lambda: ops.relu_bwd_colsum_(dh, h, db4))
        report(f"relu_bwd_colsum[{tag}] bf16", us, rows * 4 * C * 6)
        xf = torch.randn(rows, C, device=dev)
        y16 = torch.empty(rows, C, device=dev, dtype=BF)
        us = timeit(lambda: ops.colsum_cast(xf, db, y16))
        report(f"colsum_cast[{tag}] f32->bf16", us, rows * C * 6)
    z = torch.randn(R * R, cz, device=dev).to(BF)
    g, b = torch.ones(cz, device=dev), torch.zeros(cz, device=dev)
    w = torch.randn(cz, H, device=dev) * 0.1
    for swap in (False, True):
        us = timeit(lambda: ops.pair_bias_fwd(z, g, b, w, R, H, swap))
        report(f"pair_bias_fwd bf16 swap={int(swap)}", us, R * R * cz * 2 + H * R * R * 2 + R * R * 8)
    nb, mean, rstd = ops.pair_bias_fwd(z, g, b, w, R, H, False)
    dnb = torch.randn(H, R, R, device=dev)
    dz = torch.zeros(R * R, cz, device=dev)
    dw = torch.empty(cz, H, device=dev)
    us = timeit(lambda: ops.pair_bias_bwd(z, mean, rstd, g, b, w, dnb, False, dz, g.clone(), b.clone(), dw,
                                          R, H))
    report("pair_bias_bwd bf16 (dz f32 rmw)", us, R * R * cz * (2 + 8) + H * R * R * 4 + R * R * 8)
    a = torch.empty(1 << 28, dtype=torch.uint8, device=dev)
    bb = torch.empty_like(a)
    us = timeit(lambda: bb.copy_(a))
    report("torch copy 256 MB (reference)", us, 2 * a.numel())


if __name__ == "__main__":
    main()
