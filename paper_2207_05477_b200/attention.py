"""Gated self-attention with pair bias -- the reference operator API
(src/attention.py) on the sm_100a kernels.

``gated_attention_fused(inp, p)`` keeps the reference signature
(``AttentionInput`` / ``AttentionParams``, src/attention.py:35-61) and is a
``torch.autograd.Function``: forward = merged Q|K|V|G projection + the
fused attention-core kernel (+ gate) + output projection; backward = the
hand-written closure of src/attention.py:178-221 on the same kernels.
Tensors are torch CUDA tensors; parameters may require grad.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import ContractError, DimensionError


@dataclass
class AttentionParams:
    wq: torch.Tensor  # [C, H, c]
    wk: torch.Tensor
    wv: torch.Tensor
    wg: torch.Tensor
    bg: torch.Tensor  # [H, c]
    wo: torch.Tensor  # [H, c, C]
    bo: torch.Tensor  # [C]

    @property
    def heads(self) -> int:
        return self.wq.shape[1]

    @property
    def head_dim(self) -> int:
        return self.wq.shape[2]

    def all(self):
        return [self.wq, self.wk, self.wv, self.wg, self.bg, self.wo, self.bo]


@dataclass
class AttentionInput:
    x: torch.Tensor  # [B, S, R, C]
    mask: torch.Tensor  # [B, S, R] in {0, 1}
    nonbatched_bias: torch.Tensor = None  # [H, R, R]


def _check_shapes(inp: AttentionInput, p: AttentionParams):
    """src/attention.py:64-75 (same messages)."""
    b, s, r, cdim = inp.x.shape
    if p.wq.shape[0] != cdim:
        raise DimensionError(f"x channels {cdim} vs wq {tuple(p.wq.shape)}")
    if tuple(inp.mask.shape) != (b, s, r):
        raise DimensionError(f"mask shape {tuple(inp.mask.shape)} vs x {tuple(inp.x.shape)}")
    if inp.nonbatched_bias is not None:
        h = p.heads
        if tuple(inp.nonbatched_bias.shape) != (h, r, r):
            raise DimensionError(
                f"nonbatched_bias shape {tuple(inp.nonbatched_bias.shape)}, want {(h, r, r)}")


class _GatedAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, mask, nb, wq, wk, wv, wg, bg, wo, bo, act_dtype):
        b, s, r, C = x.shape
        H, D = wq.shape[1], wq.shape[2]
        HD = H * D
        T = b * s * r
        dt = act_dtype
        x2 = x.reshape(T, C).to(dt).contiguous()
        wcat = torch.cat([w.reshape(C, HD) for w in (wq, wk, wv, wg)], dim=1).to(dt).contiguous()
        qkvg = torch.empty((T, 4 * HD), dtype=dt, device=x.device)
        ops.gemm(x2, wcat, qkvg)
        maskf = mask.reshape(b * s, r).to(torch.float32).contiguous()
        bias_t = nb.to(dt).contiguous() if nb is not None else None
        bgf = bg.reshape(-1).float().contiguous()
        c_, g_, gd, lse = ops.attn_fwd(qkvg, maskf, r, 1, bias_t, bgf, b * s, r, H, D, r, 1)
        wo2 = wo.reshape(HD, C).to(dt).contiguous()
        y = torch.empty((T, C), dtype=torch.float32, device=x.device)
        ops.gemm(gd, wo2, y)
        out = torch.empty((T, C), dtype=torch.float32, device=x.device)
        ops.bias_residual(None, y, bo.float().contiguous(), out)
        ctx.save_for_backward(x2, maskf, bias_t, wcat, wo2, qkvg, c_, g_, gd, lse, bgf)
        ctx.dims = (b, s, r, C, H, D)
        ctx.has_bias = nb is not None
        return out.view(b, s, r, C)

    @staticmethod
    def backward(ctx, gout):
        x2, maskf, bias_t, wcat, wo2, qkvg, c_, g_, gd, lse, bgf = ctx.saved_tensors
        b, s, r, C, H, D = ctx.dims
        HD = H * D
        T = b * s * r
        dt = x2.dtype
        dev = x2.device
        g2 = gout.reshape(T, C).float().contiguous()
        d_act = torch.empty((T, C), dtype=dt, device=dev)
        dbo = torch.empty(C, dtype=torch.float32, device=dev)
        ops.colsum_cast(g2, dbo, y=d_act)
        dwo = torch.empty((HD, C), dtype=torch.float32, device=dev)
        ops.gemm(gd, d_act, dwo, ta=True)
        dgated = torch.empty((T, HD), dtype=dt, device=dev)
        ops.gemm(d_act, wo2, dgated, tb=True)
        dbg = torch.empty(HD, dtype=torch.float32, device=dev)
        dqkvg, dbias_t = ops.attn_bwd(qkvg, maskf, r, 1, bias_t, c_, g_, dgated, lse, dbg,
                                      b * s, r, H, D, r, 1, want_dbias=ctx.has_bias)
        dwcat = torch.empty((C, 4 * HD), dtype=torch.float32, device=dev)
        ops.gemm(x2, dqkvg, dwcat, ta=True)
        dx = torch.empty((T, C), dtype=torch.float32, device=dev)
        ops.gemm(dqkvg, wcat, dx, tb=True)
        dws = [dwcat[:, i * HD:(i + 1) * HD].reshape(C, H, D) for i in range(4)]
        dnb = dbias_t if ctx.has_bias else None
        return (dx.view(b, s, r, C), None, dnb, *dws, dbg.view(H, D), dwo.view(H, D, C), dbo, None)


def gated_attention_fused(inp: AttentionInput, p: AttentionParams,
                          act_dtype=torch.float32) -> torch.Tensor:
    """src/attention.py:118-233 -- one coarse op on the sm_100a kernels."""
    _check_shapes(inp, p)
    return _GatedAttention.apply(inp.x, inp.mask, inp.nonbatched_bias, *p.all(), act_dtype)


class _ReferenceAttention(torch.autograd.Function):
    """src/attention.py:78-115, the unfused baseline on the library's fp32
    kernels: q/k/v/gate projections, per-head logits materialised as
    [B*S, H, R, R] (q scaled before the product, :93), mask bias and pair bias
    added, softmax, context, gate, output projection -- each a separate GEMM
    or elementwise kernel; the backward is the same chain reversed."""

    @staticmethod
    def forward(ctx, x, mask, nb, wq, wk, wv, wg, bg, wo, bo):
        b, s, r, C = x.shape
        H, D = wq.shape[1], wq.shape[2]
        HD, T, BS = H * D, b * s * r, b * s
        dev, f32 = x.device, torch.float32
        x2 = x.reshape(T, C).float().contiguous()
        ws = [w.reshape(C, HD).float().contiguous() for w in (wq, wk, wv, wg)]
        scale = float(1.0 / np.sqrt(D))
        q, k, v = (torch.empty((T, HD), dtype=f32, device=dev) for _ in range(3))
        ops.gemm(x2, ws[0], q, alpha=scale)
        ops.gemm(x2, ws[1], k)
        ops.gemm(x2, ws[2], v)
        w = torch.empty((BS, H, r, r), dtype=f32, device=dev)          # logits, then weights
        for h in range(H):
            cs = slice(h * D, (h + 1) * D)
            ops.gemm_batched(q[:r, cs], k[:r, cs], w[0, h], BS, r * HD, r * HD, H * r * r, tb=True)
        maskf = mask.reshape(BS, r).float().contiguous()
        nbf = nb.float().contiguous() if nb is not None else None
        ops.softmax_masked_rows(w, maskf, r, 1, nbf, BS, H, r)
        ctx_ = torch.empty((T, HD), dtype=f32, device=dev)
        for h in range(H):
            cs = slice(h * D, (h + 1) * D)
            ops.gemm_batched(w[0, h], v[:r, cs], ctx_[:r, cs], BS, H * r * r, r * HD, r * HD)
        gp = torch.empty((T, HD), dtype=f32, device=dev)
        ops.gemm_bias(x2, ws[3], gp, bg.reshape(HD).float().contiguous())
        gate = torch.empty_like(gp)
        gated = torch.empty_like(gp)
        ops.gate_fwd(gp, ctx_, gate, gated)
        wo2 = wo.reshape(HD, C).float().contiguous()
        out = torch.empty((T, C), dtype=f32, device=dev)
        ops.gemm_bias(gated, wo2, out, bo.float().contiguous())
        ctx.save_for_backward(x2, q, k, v, w, ctx_, gate, gated, wo2, *ws)
        ctx.dims = (b, s, r, C, H, D)
        ctx.has_bias = nb is not None
        return out.view(b, s, r, C)

    @staticmethod
    def backward(ctx, gout):
        x2, q, k, v, w, ctx_, gate, gated, wo2, wq2, wk2, wv2, wg2 = ctx.saved_tensors
        b, s, r, C, H, D = ctx.dims
        HD, T, BS = H * D, b * s * r, b * s
        dev, f32 = x2.device, torch.float32
        scale = float(1.0 / np.sqrt(D))
        g2 = gout.reshape(T, C).float().contiguous()
        dbo = ops.sum_rows(g2, torch.empty(C, dtype=f32, device=dev))
        dwo = torch.empty((HD, C), dtype=f32, device=dev)
        ops.gemm(gated, g2, dwo, ta=True)
        dgated = torch.empty((T, HD), dtype=f32, device=dev)
        ops.gemm(g2, wo2, dgated, tb=True)
        dctx, dgp = torch.empty_like(dgated), torch.empty_like(dgated)
        ops.gate_bwd(dgated, gate, ctx_, dctx, dgp)
        dw = torch.empty_like(w)
        dv = torch.empty((T, HD), dtype=f32, device=dev)
        for h in range(H):
            cs = slice(h * D, (h + 1) * D)
            ops.gemm_batched(dctx[:r, cs], v[:r, cs], dw[0, h], BS, r * HD, r * HD, H * r * r, tb=True)
            ops.gemm_batched(w[0, h], dctx[:r, cs], dv[:r, cs], BS, H * r * r, r * HD, r * HD, ta=True)
        ops.softmax_rows_bwd(w, dw, BS * H * r, r)                        # dw -> d(logits)
        dnb = None
        if ctx.has_bias:
            dnb = ops.sum_rows(dw.view(BS, H * r * r), torch.empty(H * r * r, dtype=f32, device=dev)).view(H, r, r)
        dq, dk = torch.empty_like(dv), torch.empty_like(dv)           # dq: d(scaled q)
        for h in range(H):
            cs = slice(h * D, (h + 1) * D)
            ops.gemm_batched(dw[0, h], k[:r, cs], dq[:r, cs], BS, H * r * r, r * HD, r * HD)
            ops.gemm_batched(dw[0, h], q[:r, cs], dk[:r, cs], BS, H * r * r, r * HD, r * HD, ta=True)
        dws = [torch.empty((C, HD), dtype=f32, device=dev) for _ in range(4)]
        ops.gemm(x2, dq, dws[0], ta=True, alpha=scale)
        ops.gemm(x2, dk, dws[1], ta=True)
        ops.gemm(x2, dv, dws[2], ta=True)
        ops.gemm(x2, dgp, dws[3], ta=True)
        dbg = ops.sum_rows(dgp, torch.empty(HD, dtype=f32, device=dev))
        dx = torch.empty((T, C), dtype=f32, device=dev)
        ops.gemm(dq, wq2, dx, tb=True, alpha=scale)
        for dgr, wr in ((dk, wk2), (dv, wv2), (dgp, wg2)):
            ops.gemm(dgr, wr, dx, tb=True, beta=1.0)
        return (dx.view(b, s, r, C), None, dnb, *[d.view(C, H, D) for d in dws], dbg.view(H, D),
                dwo.view(H, D, C), dbo)


def gated_attention_reference(inp: AttentionInput, p: AttentionParams) -> torch.Tensor:
    """src/attention.py:78-115 -- the unfused fp32 baseline (materialised
    logits), the reference's oracle for ``gated_attention_fused``."""
    _check_shapes(inp, p)
    return _ReferenceAttention.apply(inp.x, inp.mask, inp.nonbatched_bias, *p.all())


def subbatch_apply(f, x: torch.Tensor, dim: int, chunk: int, companions=()):
    """src/attention.py:236-267: apply ``f`` over sequential chunks of ``x``
    along a batch-like ``dim`` (ragged last chunk allowed) and concatenate."""
    if chunk < 1:
        raise ContractError("chunk must be >= 1")
    extent = x.shape[dim]
    if chunk >= extent and not companions:
        return f(x)
    xs = torch.split(x, chunk, dim)
    comps = [torch.split(c, chunk, dim) for c in companions]
    outs = [f(xc, *[cc[i] for cc in comps]) for i, xc in enumerate(xs)]
    return outs[0] if len(outs) == 1 else torch.cat(outs, dim)
