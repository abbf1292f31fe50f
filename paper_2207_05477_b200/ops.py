"""Tensor-level wrappers over the C ABI.  PyTorch provides device memory and
the current stream; every byte of arithmetic runs in libevoformer_sm100.so.
"""

from __future__ import annotations

import torch

from . import _lib
from ._lib import BF16, F32, call

_DT = {torch.float32: F32, torch.bfloat16: BF16}


def dcode(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype}") from None


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t):
    return None if t is None else t.data_ptr()


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


def defer_begin(arena: torch.Tensor):
    call("evo_defer_begin", ptr(arena), arena.numel() * arena.element_size())


def defer_end(stream_obj=None):
    call("evo_defer_end", stream_obj.cuda_stream if stream_obj is not None else stream())


class deferred_reductions:
    """Context manager: batch the finalisation of every column reduction
    issued inside into one launch at exit (evo_defer_begin / evo_defer_end)."""

    def __init__(self, arena: torch.Tensor):
        self.arena = arena

    def __enter__(self):
        call("evo_defer_begin", ptr(self.arena), self.arena.numel() * self.arena.element_size())
        return self

    def __exit__(self, *exc):
        call("evo_defer_end", stream())
        return False


# ---------------------------------------------------------------------------
# GEMM


def gemm(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, ta: bool = False, tb: bool = False,
         alpha: float = 1.0, beta: float = 0.0):
    """c = alpha * op(a) @ op(b) + beta * c for row-major 2-D (possibly
    column-sliced) views with unit inner stride."""
    for t in (a, b, c):
        if t.dim() != 2 or t.stride(1) != 1:
            raise ValueError("gemm operands must be 2-D with unit inner stride")
    M, K = (a.shape[1], a.shape[0]) if ta else (a.shape[0], a.shape[1])
    Kb, N = (b.shape[1], b.shape[0]) if tb else (b.shape[0], b.shape[1])
    if K != Kb or tuple(c.shape) != (M, N):
        raise ValueError(f"gemm shape mismatch: op(a)={M}x{K} op(b)={Kb}x{N} c={tuple(c.shape)}")
    if a.dtype != b.dtype:
        raise TypeError("gemm: a and b must share a dtype")
    call("evo_gemm", M, N, K, ptr(a), a.stride(0), int(ta), 0, ptr(b), b.stride(0), int(tb), 0,
         ptr(c), c.stride(0), 0, 1, alpha, beta, dcode(a), dcode(c), stream())


def gemm_bias(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, bias: torch.Tensor,
              res: torch.Tensor | None = None, relu: bool = False, ta: bool = False, tb: bool = False,
              bias16: torch.Tensor | None = None):
    """out = op(a) @ op(b) + bias (+ res), or relu(op(a) @ op(b) + bias): the
    projection with its module epilogue fused (one kernel on the Lt path)."""
    for t in (a, b, out):
        if t.dim() != 2 or t.stride(1) != 1:
            raise ValueError("gemm operands must be 2-D with unit inner stride")
    M, K = (a.shape[1], a.shape[0]) if ta else (a.shape[0], a.shape[1])
    Kb, N = (b.shape[1], b.shape[0]) if tb else (b.shape[0], b.shape[1])
    if K != Kb or tuple(out.shape) != (M, N) or bias.numel() != N:
        raise ValueError(f"gemm_bias shape mismatch: op(a)={M}x{K} op(b)={Kb}x{N} out={tuple(out.shape)}")
    if res is not None and (tuple(res.shape) != (M, N) or not res.is_contiguous() or not out.is_contiguous()):
        raise ValueError("gemm_bias: residual must be a contiguous [M, N] like out")
    if bias16 is not None and bias16.dtype != torch.bfloat16:
        bias16 = None
    call("evo_gemm_bias", M, N, K, ptr(a), a.stride(0), int(ta), ptr(b), b.stride(0), int(tb), ptr(res),
         dcode(res) if res is not None else F32, ptr(bias), ptr(bias16), int(relu), ptr(out), out.stride(0),
         dcode(a), dcode(out), stream())
    return out


def gemm_relu_mask(a, b, h, out, ta=False, tb=False, colsum=None, accumulate=False):
    """out = (h > 0) * (op(a) @ op(b)): the ReLU backward fused into the
    d(hidden) GEMM's epilogue (bf16 only); with ``colsum`` (fp32 [N]) the
    epilogue also writes the column sums of ``out`` (the hidden bias
    gradient)."""
    M, K = (a.shape[1], a.shape[0]) if ta else (a.shape[0], a.shape[1])
    Kb, N = (b.shape[1], b.shape[0]) if tb else (b.shape[0], b.shape[1])
    if K != Kb or tuple(out.shape) != (M, N) or tuple(h.shape) != (M, N):
        raise ValueError("gemm_relu_mask shape mismatch")
    if not (h.is_contiguous() and out.is_contiguous()):
        raise ValueError("gemm_relu_mask: h and out must be contiguous")
    ws = _ws(_lib.load().evo_gemm_relu_mask_workspace(M, N), out.device) if colsum is not None else None
    call("evo_gemm_relu_mask", M, N, K, ptr(a), a.stride(0), int(ta), ptr(b), b.stride(0), int(tb), ptr(h),
         ptr(out), dcode(out), ptr(colsum), int(accumulate), ptr(ws), stream())
    return out


def gemm_batched(a, b, c, batch, sa, sb, sc, ta=False, tb=False, alpha=1.0, beta=0.0):
    """Strided-batched row-major GEMM on flat buffers: operand k of batch i is
    the matrix at data_ptr + i*s (elements); a, b, c are 2-D views of batch 0."""
    M, K = (a.shape[1], a.shape[0]) if ta else (a.shape[0], a.shape[1])
    Kb, N = (b.shape[1], b.shape[0]) if tb else (b.shape[0], b.shape[1])
    if K != Kb or tuple(c.shape) != (M, N):
        raise ValueError("gemm_batched shape mismatch")
    call("evo_gemm", M, N, K, ptr(a), a.stride(0), int(ta), sa, ptr(b), b.stride(0), int(tb), sb,
         ptr(c), c.stride(0), sc, batch, alpha, beta, dcode(a), dcode(c), stream())


# ---------------------------------------------------------------------------
# triangle multiplication glue


def trimul_gate_fwd(proj, biases, mask, ch):
    RR = proj.shape[0]
    a = torch.empty((ch, RR), dtype=proj.dtype, device=proj.device)
    b = torch.empty_like(a)
    call("evo_trimul_gate_fwd", ptr(proj), proj.stride(0), *[ptr(t) for t in biases], ptr(mask),
         ptr(a), ptr(b), RR, ch, dcode(proj), stream())
    return a, b


def trimul_gate_bwd(proj, biases, mask, da, db, ch):
    RR = proj.shape[0]
    dproj = torch.empty((RR, 4 * ch), dtype=proj.dtype, device=proj.device)
    call("evo_trimul_gate_bwd", ptr(proj), proj.stride(0), *[ptr(t) for t in biases], ptr(mask),
         ptr(da), ptr(db), ptr(dproj), RR, ch, dcode(proj), stream())
    return dproj


def transpose2d(x, out_dtype=None):
    rows, cols = x.shape
    y = torch.empty((cols, rows), dtype=out_dtype or x.dtype, device=x.device)
    call("evo_transpose2d", ptr(x), dcode(x), ptr(y), dcode(y), rows, cols, stream())
    return y


def gated_residual(res, gp, bg, y, by):
    rows, C = y.shape
    g = torch.empty_like(y)
    out = torch.empty_like(y)
    call("evo_gated_residual", ptr(res), ptr(gp), gp.stride(0), ptr(bg), ptr(y), ptr(by), ptr(g),
         ptr(out), rows, C, dcode(y), stream())
    return g, out


def gated_residual_bwd(dout, g, y, by):
    rows, C = y.shape
    dyb = torch.empty_like(y)
    dgp = torch.empty_like(y)
    call("evo_gated_residual_bwd", ptr(dout), ptr(g), ptr(y), ptr(by), ptr(dyb), ptr(dgp), rows, C,
         dcode(y), stream())
    return dyb, dgp


# ---------------------------------------------------------------------------
# LayerNorm / glue


def layernorm(x: torch.Tensor, g: torch.Tensor, b: torch.Tensor, out_dtype, eps: float = 1e-5):
    rows, C = x.shape
    y = torch.empty((rows, C), dtype=out_dtype, device=x.device)
    mean = torch.empty(rows, dtype=torch.float32, device=x.device)
    rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
    call("evo_layernorm_fwd", ptr(x), dcode(x), ptr(g), ptr(b), ptr(y), dcode(y), ptr(mean),
         ptr(rstd), rows, C, eps, stream())
    return y, mean, rstd


def layernorm_bwd(x, dy, mean, rstd, g, dres, dx, dgamma, dbeta, accumulate=False):
    rows, C = x.shape
    ws = _ws(_lib.load().evo_layernorm_bwd_workspace(rows, C), x.device)
    call("evo_layernorm_bwd", ptr(x), dcode(x), ptr(dy), dcode(dy), ptr(mean), ptr(rstd), ptr(g),
         ptr(dres), ptr(dx), ptr(dgamma), ptr(dbeta), int(accumulate), ptr(ws), rows, C, stream())


def layernorm_bwd_ex(x, dy, mean, rstd, g, dres, dx, dgamma, dbeta, dx16, dxsum, accumulate=False):
    """layernorm_bwd that also emits a bf16 copy of dx and its column sums:
    the next module's GEMM operand and output-bias gradient in the same pass."""
    rows, C = x.shape
    ws = _ws(_lib.load().evo_layernorm_bwd_workspace(rows, C), x.device)
    call("evo_layernorm_bwd_ex", ptr(x), dcode(x), ptr(dy), dcode(dy), ptr(mean), ptr(rstd), ptr(g),
         ptr(dres), ptr(dx), ptr(dx16), ptr(dxsum), ptr(dgamma), ptr(dbeta), int(accumulate), ptr(ws), rows,
         C, stream())


def bias_residual(res, y, bias, out):
    rows, C = y.shape
    call("evo_bias_residual", ptr(res), dcode(res) if res is not None else F32, ptr(y), dcode(y),
         ptr(bias), ptr(out), dcode(out), rows, C, stream())
    return out


def bias_relu_(y, bias):
    rows, C = y.shape
    call("evo_bias_relu", ptr(y), dcode(y), ptr(bias), rows, C, stream())


def relu_bwd_colsum_(dh, h, db, accumulate=False):
    rows, C = dh.shape
    ws = _ws(_lib.load().evo_colsum_workspace(C), dh.device)
    call("evo_relu_bwd_colsum", ptr(dh), ptr(h), dcode(dh), ptr(db), int(accumulate), ptr(ws),
         rows, C, stream())


def colsum_cast(x, out, y=None, accumulate=False):
    rows, C = x.shape
    ws = _ws(_lib.load().evo_colsum_workspace(C), x.device)
    call("evo_colsum_cast", ptr(x), dcode(x), ptr(out), int(accumulate), ptr(y),
         dcode(y) if y is not None else F32, ptr(ws), rows, C, stream())


def colsum_strided(x, out, accumulate=False):
    """Column sums of a 2-D view whose rows are strided (a column slice)."""
    rows, C = x.shape
    assert x.stride(1) == 1
    ws = _ws(_lib.load().evo_colsum_workspace(C), x.device)
    call("evo_colsum_strided", ptr(x), dcode(x), x.stride(0), ptr(out), int(accumulate), ptr(ws),
         rows, C, stream())


class PackPlan:
    """Host-side pointer tables for evo_pack_cols (built once: the pooled
    parameter storage and the packed buffers never move)."""

    def __init__(self, srcs, dsts, Cs, Ns, unpack, sdt, ddt, ns=4):
        import ctypes
        P = ctypes.c_void_p
        self.src = (P * len(srcs))(*[t.data_ptr() for t in srcs])
        self.dst = (P * len(dsts))(*[t.data_ptr() for t in dsts])
        self.C = (ctypes.c_int64 * len(Cs))(*Cs)
        self.N = (ctypes.c_int64 * len(Ns))(*Ns)
        self.n = len(Cs)
        self.unpack, self.sdt, self.ddt, self.ns = int(unpack), sdt, ddt, int(ns)
        self.keep = (srcs, dsts)

    def run(self):
        call("evo_pack_cols_ns", self.src, self.dst, self.C, self.N, self.n, self.ns, self.sdt, self.ddt,
             self.unpack, stream())


def scale_(y, s):
    """y *= s in place (fp32)."""
    call("evo_scale_inplace", ptr(y), float(s), y.numel(), stream())
    return y


def cast(x, y):
    call("evo_cast", ptr(x), dcode(x), ptr(y), dcode(y), x.numel(), stream())
    return y


# ---------------------------------------------------------------------------
# attention core


# -- unfused attention baseline pieces (gated_attention_reference) ----------


def softmax_masked_rows(x, mask, msb, msl, nb, BS, H, R):
    """In place on fp32 logits [BS, H, R, R]: softmax_j(x + (mask - 1) * 1e9 + nb)."""
    call("evo_softmax_masked_rows", ptr(x), ptr(mask), msb, msl, ptr(nb), BS, H, R, stream())


def softmax_rows_bwd(w, g, rows, R):
    call("evo_softmax_rows_bwd", ptr(w), ptr(g), rows, R, stream())


def gate_fwd(gp, ctx, gate, gated):
    call("evo_gate_fwd", ptr(gp), ptr(ctx), ptr(gate), ptr(gated), gp.numel(), stream())


def gate_bwd(dgated, gate, ctx, dctx, dgp):
    call("evo_gate_bwd", ptr(dgated), ptr(gate), ptr(ctx), ptr(dctx), ptr(dgp), dgated.numel(), stream())


def sum_rows(x, out, accumulate=False):
    rows, cols = x.shape
    call("evo_sum_rows", ptr(x), rows, cols, ptr(out), int(accumulate), stream())
    return out


def attn_fwd(qkvg, mask, msb, msl, nb, bg, B, L, H, D, sb, sl):
    """nb: [H, L, L] (query, key) in qkvg's dtype, or None."""
    T = qkvg.shape[0]
    dev, dt = qkvg.device, qkvg.dtype
    if nb is not None and nb.dtype != dt:
        raise TypeError("attention bias must be stored in the activation dtype")
    ctx = torch.empty((T, H * D), dtype=dt, device=dev)
    gate = torch.empty_like(ctx)
    gated = torch.empty_like(ctx)
    lse = torch.empty((B, H, L, 2), dtype=torch.float32, device=dev)
    call("evo_attn_fwd", ptr(qkvg), qkvg.stride(0), ptr(mask), msb, msl, ptr(nb), ptr(bg),
         ptr(ctx), ptr(gate), ptr(gated), ptr(lse), B, L, H, D, sb, sl, dcode(qkvg), stream())
    return ctx, gate, gated, lse


def attn_bwd(qkvg, mask, msb, msl, nb, ctx, gate, dgated, lse, dbg, B, L, H, D, sb, sl,
             want_dbias: bool, accumulate=False):
    """Returns (dqkvg, dnb [H, L, L] fp32 or None)."""
    dev = qkvg.device
    dqkvg = torch.empty_like(qkvg)
    dnb = torch.empty((H, L, L), dtype=torch.float32, device=dev) if want_dbias else None
    nbytes = _lib.load().evo_attn_bwd_workspace(B, L, H, D, dcode(qkvg))
    ws = _ws(nbytes, dev)
    call("evo_attn_bwd", ptr(qkvg), qkvg.stride(0), ptr(mask), msb, msl, ptr(nb), ptr(ctx),
         ptr(gate), ptr(dgated), ptr(lse), ptr(dqkvg), ptr(dnb), ptr(dbg), int(accumulate),
         ptr(ws), ws.numel(), B, L, H, D, sb, sl, dcode(qkvg), stream())
    return dqkvg, dnb


# ---------------------------------------------------------------------------
# pair bias


def pair_bias_fwd(z, g, b, w, R, H, swap_xy, ni=None, nj=None):
    """nb [H, R, R] (query, key) in z's dtype; swap_xy for triangle-end.  With
    (ni, nj) z holds an ni x nj token block (a DAP shard) and nb is
    [H, ni, nj] (or [H, nj, ni] with swap_xy)."""
    C = z.shape[1]
    dev = z.device
    ni = R if ni is None else ni
    nj = R if nj is None else nj
    nb = torch.empty((H, nj, ni) if swap_xy else (H, ni, nj), dtype=z.dtype, device=dev)
    mean = torch.empty(ni * nj, dtype=torch.float32, device=dev)
    rstd = torch.empty(ni * nj, dtype=torch.float32, device=dev)
    call("evo_pair_bias_fwd_rect", ptr(z), dcode(z), ptr(g), ptr(b), ptr(w), ptr(nb), ptr(mean),
         ptr(rstd), ni, nj, C, H, int(swap_xy), stream())
    return nb, mean, rstd


def ln_pair_bias_fwd(z, lg, lb, g, b, w, R, H, swap_xy, ni=None, nj=None):
    """One pass over the pair rows z for the triangle attentions: their input
    LayerNorm (lg, lb) -> xl (bf16) and the pair bias nb as pair_bias_fwd, with
    the shared row statistics.  Returns (xl, nb, mean, rstd), or None when the
    fused kernel does not cover the shape (bf16, c_z = 128, H <= 8, >= 4096
    rows) -- the caller then runs layernorm + pair_bias_fwd."""
    C = z.shape[1]
    ni = R if ni is None else ni
    nj = R if nj is None else nj
    if z.dtype != torch.bfloat16 or C != 128 or H > 8 or ni * nj < 4096 or not z.is_contiguous():
        return None
    dev = z.device
    xl = torch.empty_like(z)
    nb = torch.empty((H, nj, ni) if swap_xy else (H, ni, nj), dtype=z.dtype, device=dev)
    mean = torch.empty(ni * nj, dtype=torch.float32, device=dev)
    rstd = torch.empty(ni * nj, dtype=torch.float32, device=dev)
    call("evo_ln_pair_bias_fwd", ptr(z), dcode(z), ptr(lg), ptr(lb), ptr(g), ptr(b), ptr(w), ptr(xl), ptr(nb),
         ptr(mean), ptr(rstd), ni, nj, C, H, int(swap_xy), stream())
    return xl, nb, mean, rstd


def pair_bias_bwd(z, mean, rstd, g, b, w, dnb, swap_xy, dz, dg, db, dw, R, H,
                  accumulate=False, ni=None, nj=None, dz16=None, dzsum=None):
    """With ``dz16`` / ``dzsum`` the pass also emits the updated dz as bf16
    and its column sums (the next module's operand and output-bias gradient);
    shapes the fused path does not cover get a separate colsum/cast pass."""
    C = z.shape[1]
    ni = R if ni is None else ni
    nj = R if nj is None else nj
    ws = _ws(_lib.load().evo_pair_bias_bwd_workspace(C, H), z.device)
    fused_ok = (z.dtype == torch.bfloat16 and C == 128 and H <= 8 and (ni * nj) % 4 == 0 and ni * nj >= 4096)
    if (dz16 is not None or dzsum is not None) and fused_ok:
        call("evo_pair_bias_bwd_ex", ptr(z), dcode(z), ptr(mean), ptr(rstd), ptr(g), ptr(b), ptr(w),
             ptr(dnb), int(swap_xy), ptr(dz), ptr(dg), ptr(db), ptr(dw), int(accumulate),
             ptr(ws), ni, nj, C, H, ptr(dz16), ptr(dzsum), stream())
        return
    call("evo_pair_bias_bwd_rect", ptr(z), dcode(z), ptr(mean), ptr(rstd), ptr(g), ptr(b), ptr(w),
         ptr(dnb), int(swap_xy), ptr(dz), ptr(dg), ptr(db), ptr(dw), int(accumulate),
         ptr(ws), ni, nj, C, H, stream())
    if dz16 is not None or dzsum is not None:
        colsum_cast(dz, dzsum, y=dz16)


# ---------------------------------------------------------------------------
# outer product mean


def opm_proj(ab, bl, br, mask_flat, k):
    SR = ab.shape[0]
    a = torch.empty((SR, k), dtype=ab.dtype, device=ab.device)
    c = torch.empty_like(a)
    call("evo_opm_proj", ptr(ab), ptr(bl), ptr(br), ptr(mask_flat), ptr(a), ptr(c), SR, k,
         dcode(ab), stream())
    return a, c


def opm_proj_bwd(da, dc, mask_flat, dbl, dbr, k, accumulate=False):
    SR = mask_flat.numel()
    d_ab = torch.empty((SR, 2 * k), dtype=da.dtype, device=da.device)
    ws = _ws(_lib.load().evo_colsum_workspace(2 * k), da.device)
    call("evo_opm_proj_bwd", ptr(da), ptr(dc), ptr(mask_flat), ptr(d_ab), ptr(dbl), ptr(dbr),
         int(accumulate), ptr(ws), SR, k, dcode(da), stream())
    return d_ab


def opm_rec(mask, S, R, i0=0, ni=None):
    """rec rows i0..i0+ni-1 = 1 / (mask^T mask + 1e-3): a function of the mask only."""
    ni = R if ni is None else ni
    rec = torch.empty(ni * R, dtype=torch.float32, device=mask.device)
    call("evo_opm_rec", ptr(mask), ptr(rec), S, R, i0, ni, stream())
    return rec


def opm_norm_fwd(num, mask, S, R, k, out_dtype, i0=0, ni=None, rec=None):
    """num holds rows i0..i0+ni-1 (all R rows by default; a DAP shard otherwise).
    With ``rec`` (from opm_rec) only the normalisation runs."""
    dev = num.device
    ni = R if ni is None else ni
    if rec is not None:
        outn = torch.empty((ni * R, k * k), dtype=out_dtype, device=dev)
        call("evo_opm_norm_apply_rows", ptr(num), dcode(num), ptr(rec), ptr(outn), dcode(outn), R, k, ni,
             stream())
        return rec, outn
    rec = torch.empty(ni * R, dtype=torch.float32, device=dev)
    outn = torch.empty((ni * R, k * k), dtype=out_dtype, device=dev)
    call("evo_opm_norm_fwd_rows", ptr(num), dcode(num), ptr(mask), ptr(rec), ptr(outn), dcode(outn),
         S, R, k, i0, ni, stream())
    return rec, outn


def opm_dnum(d_act, w_out, rec, R, k, ni=None):
    """d(num) straight from d(pair): the w_out data-gradient GEMM with the OPM
    normalisation and re-layout in its tcgen05 epilogue (gemm_tc.cu OPM mode).  None when the shape
    is not covered (the caller runs GEMM + opm_norm_bwd)."""
    ni = R if ni is None else ni
    C = d_act.shape[1]
    if (d_act.dtype != torch.bfloat16 or w_out.dtype != torch.bfloat16 or C % 8 or k != 32
            or R % 128 or not d_act.is_contiguous() or not w_out.is_contiguous()):
        return None
    dnum = torch.empty((ni * k, R * k), dtype=torch.bfloat16, device=d_act.device)
    call("evo_opm_dnum", ptr(d_act), ptr(w_out), ptr(rec), ptr(dnum), R, k, ni, C, dcode(d_act), stream())
    return dnum


def opm_outn(a, c, rec, S, R, k, ni=None):
    """The OPM's normalised outer-product block outn [(i, j), p*k+q] straight
    from the projections a, c [S, R*k]: the sum over sequences as one tcgen05
    GEMM with the normalisation and re-layout in its epilogue.  None when the
    shape is not covered (the caller runs GEMM + opm_norm_fwd)."""
    ni = R if ni is None else ni
    if (a.dtype != torch.bfloat16 or c.dtype != torch.bfloat16 or S % 8 or k != 32 or ni != R
            or not a.is_contiguous() or not c.is_contiguous()):
        return None
    outn = torch.empty((ni * R, k * k), dtype=torch.bfloat16, device=a.device)
    call("evo_opm_outn", ptr(a), ptr(c), ptr(rec), ptr(outn), S, R, k, ni, dcode(a), stream())
    return outn


def opm_norm_bwd(doutn, rec, R, k, out_dtype, ni=None):
    ni = R if ni is None else ni
    dnum = torch.empty((ni * k, R * k), dtype=out_dtype, device=doutn.device)
    call("evo_opm_norm_bwd_rows", ptr(doutn), dcode(doutn), ptr(rec), ptr(dnum), dcode(dnum), R, k,
         ni, stream())
    return dnum


def swap01(src, A, B, out=None):
    """out[b, a, ...] = src[a, b, ...] for src viewed as [A, B, rest] (contiguous)."""
    if not src.is_contiguous():
        raise ValueError("swap01: src must be contiguous")
    n = src.numel()
    if n % (A * B):
        raise ValueError(f"swap01: {n} elements do not split into {A} x {B} rows")
    out = torch.empty_like(src) if out is None else out
    call("evo_swap01", ptr(src), ptr(out), A, B, (n // (A * B)) * src.element_size(), stream())
    return out


# ---------------------------------------------------------------------------
# loss and optimizer


def sq_loss(msa, pair, km, kz):
    dev = msa.device
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    dmsa = torch.empty(msa.shape, dtype=torch.float32, device=dev)
    dpair = torch.empty(pair.shape, dtype=torch.float32, device=dev)
    ws = _ws(_lib.load().evo_sq_loss_workspace(), dev)
    call("evo_sq_loss", ptr(msa), msa.numel(), ptr(pair), pair.numel(), dcode(msa), km, kz,
         ptr(loss), ptr(dmsa), ptr(dpair), ptr(ws), stream())
    return loss, dmsa, dpair


def sumsq_f64(g, out):
    ws = _ws(_lib.load().evo_sumsq_workspace(), g.device)
    call("evo_sumsq_f64", ptr(g), g.numel(), ptr(out), ptr(ws), stream())


def adam_clip_ema(p, g, m, v, ema, p_bf16, sumsq, clip, lr, b1, omb1, b2, omb2, eps, bc1, bc2,
                  decay, omdecay):
    call("evo_adam_clip_ema", ptr(p), ptr(g), ptr(m), ptr(v), ptr(ema), ptr(p_bf16), p.numel(),
         ptr(sumsq), clip, lr, b1, omb1, b2, omb2, eps, bc1, bc2, decay, omdecay, stream())


def sumsq_f64_step(g, out, step, bc_table, bc_out):
    ws = _ws(_lib.load().evo_sumsq_workspace(), g.device)
    call("evo_sumsq_f64_step", ptr(g), g.numel(), ptr(out), ptr(ws), ptr(step), ptr(bc_table),
         bc_table.shape[1], ptr(bc_out), stream())


def adam_clip_ema_dev(p, g, m, v, ema, p_bf16, sumsq, clip, lr, b1, omb1, b2, omb2, eps, bc, decay, omdecay):
    call("evo_adam_clip_ema_dev", ptr(p), ptr(g), ptr(m), ptr(v), ptr(ema), ptr(p_bf16), p.numel(),
         ptr(sumsq), clip, lr, b1, omb1, b2, omb2, eps, ptr(bc), decay, omdecay, stream())
