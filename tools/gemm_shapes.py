"""Record every evo_gemm call of one block fwd+bwd at the bench shape, then
time each distinct (M, N, K, ta, tb, dtypes) in isolation with CUDA events.

    python tools/gemm_shapes.py
"""
import os
import sys
from collections import Counter

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402
from paper_2207_05477_b200.model import ModelConfig  # noqa: E402
from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer  # noqa: E402


def main():
    cfg = ModelConfig(n_blocks=1, n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32)
    tr = Trainer.create(cfg, ExecutionPlan(act_dtype="bf16", fixed_recycles=1))
    tr.engine.forward_backward(tr.feats, 1)
    torch.cuda.synchronize()
    calls = []
    orig = ops.call

    def rec(name, *args):
        if name == "evo_gemm":
            M, N, K = args[0], args[1], args[2]
            ta, tb, batch = args[5], args[9], args[14]
            ad, cd = args[17], args[18]
            calls.append((M, N, K, ta, tb, batch, ad, cd, 0))
        elif name == "evo_gemm_bias":
            M, N, K = args[0], args[1], args[2]
            ta, tb = args[5], args[8]
            epi = 2 if args[13] else (3 if args[9] else 1)   # relu / residual / bias only
            calls.append((M, N, K, ta, tb, 1, args[16], args[17], epi))
        return orig(name, *args)

    ops.call = rec
    tr.engine.forward_backward(tr.feats, 1)
    ops.call = orig
    torch.cuda.synchronize()
    cnt = Counter(calls)
    dt = {0: torch.float32, 1: torch.bfloat16}
    tot_t = tot_f = tot_cb = 0.0
    rows = []
    for (M, N, K, ta, tb, batch, ad, cd, epi), n in cnt.items():
        a = torch.randn((K, M) if ta else (M, K), device="cuda").to(dt.get(ad, torch.bfloat16))
        b = torch.randn((N, K) if tb else (K, N), device="cuda").to(dt.get(ad, torch.bfloat16))
        c = torch.empty((M, N), device="cuda", dtype=dt.get(cd, torch.float32))
        if batch != 1:
            continue
        bias = torch.zeros(N, device="cuda")
        res = torch.zeros_like(c) if epi == 3 else None

        def run():
            if epi:
                ops.gemm_bias(a, b, c, bias, res=res, relu=epi == 2, ta=bool(ta), tb=bool(tb))
            else:
                ops.gemm(a, b, c, ta=bool(ta), tb=bool(tb))
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(20):
                run()
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        # cuBLAS (torch.matmul, bf16 out) on the same operands, for comparison only
        at = a.t() if ta else a
        bt = b.t() if tb else b
        for _ in range(3):
            torch.matmul(at, bt)
        gr2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr2):
            for _ in range(20):
                torch.matmul(at, bt)
        gr2.replay()
        torch.cuda.synchronize()
        e0.record()
        gr2.replay()
        e1.record()
        torch.cuda.synchronize()
        us_cublas = e0.elapsed_time(e1) / 20 * 1e3
        fl = 2.0 * M * N * K
        tot_t += us * n
        tot_f += fl * n
        es = 2 if cd == 1 else 4
        byt = (M * K + K * N) * (2 if ad == 1 else 4) + M * N * es * (2 if epi == 3 else 1)
        rows.append((us * n, M, N, K, ta, tb, ad, cd, n, us, fl / us / 1e6, epi, byt / us / 1e3, us_cublas))
        tot_cb += us_cublas * n
    for r in sorted(rows, reverse=True):
        print(f"M={r[1]:6d} N={r[2]:6d} K={r[3]:6d} ta={r[4]} tb={r[5]} a{r[6]} c{r[7]} epi{r[11]} x{r[8]}  "
              f"{r[9]:8.1f} us  {r[10]:7.1f} TF/s {r[12]:7.0f} GB/s  total {r[0]:8.1f} us  cublas {r[13]:8.1f} us")
    print(f"per block: {tot_t:.1f} us, {tot_f / tot_t / 1e6:.1f} TF/s; cublas (bf16 out) {tot_cb:.1f} us")


if __name__ == "__main__":
    main()
