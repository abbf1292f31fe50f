"""Kernel-level numerics of the sm_100a library against plain PyTorch fp32
references of the same op (floating-point kernels), for every attention
geometry the Evoformer uses (MSA row / column, triangle start / end) and the
ragged key counts the padding logic has to handle.

Tolerances: fp32 SIMT path 1e-5 relative; bf16 tensor-core path 2e-2 relative
on bf16-stored outputs (inputs are the same bf16 tensors; the differences
are the bf16 rounding of P and of the outputs)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_05477_b200 import _lib
    _lib.lib()


def rel(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).abs().max() / max(a.abs().max(), b.abs().max(), 1e-30))


def ref_attention(qkvg, mask, msb, msl, bias_t, bg, B, L, H, D, sb, sl):
    """fp32 torch reference in the reference's op order (src/attention.py:141-174)."""
    HD = H * D
    dev = qkvg.device
    b = torch.arange(B, device=dev)[:, None]
    l = torch.arange(L, device=dev)[None, :]
    tok = (b * sb + l * sl)                     # [B, L]
    x = qkvg.float()[tok]                      # [B, L, 4HD]
    q = x[..., :HD].view(B, L, H, D).transpose(1, 2)
    k = x[..., HD:2 * HD].view(B, L, H, D).transpose(1, 2)
    v = x[..., 2 * HD:3 * HD].view(B, L, H, D).transpose(1, 2)
    gp = x[..., 3 * HD:]
    m = mask[(b * msb + l * msl)]               # [B, L]
    logits = (q @ k.transpose(-1, -2)) * np.float32(1.0 / np.sqrt(D))
    logits = logits + ((m - 1.0) * 1e9)[:, None, None, :]
    if bias_t is not None:
        logits = logits + bias_t.float()[None]
    w = torch.softmax(logits, dim=-1)
    ctx = (w @ v).transpose(1, 2).reshape(B, L, HD)
    gate = torch.sigmoid(gp + bg)
    out_ctx = torch.empty(qkvg.shape[0], HD, device=dev)
    out_gate = torch.empty_like(out_ctx)
    out_ctx[tok.reshape(-1)] = ctx.reshape(-1, HD)
    out_gate[tok.reshape(-1)] = gate.reshape(-1, HD)
    return out_ctx, out_gate, w


GEOMS = {
    # name: (B, L, sb, sl, msb, msl, bias, bias_transposed_source)
    "row": lambda S, R: (S, R, R, 1, R, 1),
    "col": lambda S, R: (R, S, 1, R, 1, R),
    "tri_start": lambda S, R: (R, R, R, 1, R, 1),
    "tri_end": lambda S, R: (R, R, 1, R, 1, R),
}


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("geom", list(GEOMS))
@pytest.mark.parametrize("S,R,H,D", [(8, 32, 2, 16), (12, 40, 2, 32), (6, 64, 4, 16),
                                     (16, 100, 2, 32), (4, 256, 8, 16), (4, 256, 8, 32),
                                     (8, 200, 2, 16)])
def test_attention_fwd_vs_torch(dtype, geom, S, R, H, D):
    from paper_2207_05477_b200 import ops
    torch.manual_seed(S * 1000 + R + H + D)
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    B, L, sb, sl, msb, msl = GEOMS[geom](S, R)
    T = S * R if geom in ("row", "col") else R * R
    HD = H * D
    qkvg = (torch.randn(T, 4 * HD, device="cuda") * 0.7).to(dt)
    mask = torch.ones(T, device="cuda")
    n_valid = R - R // 10
    mv = mask.view(S, R) if geom in ("row", "col") else mask.view(R, R)
    mv[:, n_valid:] = 0.0
    if geom in ("tri_start", "tri_end"):
        mv[n_valid:, :] = 0.0
    use_bias = geom != "col"
    bias_t = (torch.randn(H, L, L, device="cuda") * 0.3).to(dt) if use_bias else None
    bg = torch.randn(HD, device="cuda") * 0.1
    ctx, gate, gated, lse = ops.attn_fwd(qkvg, mask, msb, msl, bias_t, bg, B, L, H, D, sb, sl)
    rc, rg, w = ref_attention(qkvg, mask, msb, msl, bias_t, bg, B, L, H, D, sb, sl)
    tol = 1e-5 if dtype == "f32" else 2e-2
    assert rel(ctx.float(), rc) <= tol
    assert rel(gate.float(), rg) <= tol
    assert rel(gated.float(), rc * rg) <= tol * 2
    # saved (row max, 1/row sum) reproduce the probabilities
    assert torch.isfinite(lse).all()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("geom", list(GEOMS))
@pytest.mark.parametrize("S,R,H,D", [(8, 32, 2, 16), (6, 64, 4, 16), (16, 100, 2, 32),
                                     (4, 256, 8, 16), (4, 256, 8, 32)])
def test_attention_bwd_vs_torch(dtype, geom, S, R, H, D):
    """Backward of the core (dq, dk, dv, d gate pre-activation, dbias, dbg)
    against torch autograd through the fp32 reference."""
    from paper_2207_05477_b200 import ops
    torch.manual_seed(7 * S + R + H * D)
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    B, L, sb, sl, msb, msl = GEOMS[geom](S, R)
    T = S * R if geom in ("row", "col") else R * R
    HD = H * D
    qkvg = (torch.randn(T, 4 * HD, device="cuda") * 0.7).to(dt)
    mask = torch.ones(T, device="cuda")
    n_valid = R - R // 10
    mv = mask.view(S, R) if geom in ("row", "col") else mask.view(R, R)
    mv[:, n_valid:] = 0.0
    if geom in ("tri_start", "tri_end"):
        mv[n_valid:, :] = 0.0
    use_bias = geom != "col"
    bias_t = (torch.randn(H, L, L, device="cuda") * 0.3).to(dt) if use_bias else None
    bg = torch.randn(HD, device="cuda") * 0.1
    ctx, gate, gated, lse = ops.attn_fwd(qkvg, mask, msb, msl, bias_t, bg, B, L, H, D, sb, sl)
    dgated = (torch.randn(T, HD, device="cuda") * 0.5).to(dt)
    dbg = torch.empty(HD, device="cuda")
    dqkvg, dbias_t = ops.attn_bwd(qkvg, mask, msb, msl, bias_t, ctx, gate, dgated, lse, dbg,
                                  B, L, H, D, sb, sl, want_dbias=use_bias)
    # reference gradient
    qr = qkvg.float().clone().requires_grad_(True)
    br = bias_t.float().clone().requires_grad_(True) if use_bias else None
    bgr = bg.clone().requires_grad_(True)
    rc, rg, _ = ref_attention(qr, mask, msb, msl, br, bgr, B, L, H, D, sb, sl)
    (rc * rg * dgated.float()).sum().backward()
    tol = 1e-4 if dtype == "f32" else 3e-2
    for s, name in enumerate(("dq", "dk", "dv", "dg")):
        got = dqkvg[:, s * HD:(s + 1) * HD].float()
        want = qr.grad[:, s * HD:(s + 1) * HD]
        assert rel(got, want) <= tol, name
    assert rel(dbg, bgr.grad) <= tol
    if use_bias:
        assert rel(dbias_t, br.grad) <= tol


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("C", [32, 64, 128, 256])
def test_layernorm_fwd_bwd_vs_torch(dtype, C):
    from paper_2207_05477_b200 import ops
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    torch.manual_seed(C)
    x = (torch.randn(1000, C, device="cuda") * 2 + 0.5).to(dt)
    g = torch.randn(C, device="cuda")
    b = torch.randn(C, device="cuda")
    y, mu, rs = ops.layernorm(x, g, b, dt)
    xr = x.float().requires_grad_(True)
    gr, brr = g.clone().requires_grad_(True), b.clone().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xr, (C,), gr, brr, 1e-5)
    tol = 1e-5 if dtype == "f32" else 1e-2
    assert rel(y.float(), yr) <= tol
    dy = torch.randn(1000, C, device="cuda").to(dt)
    dres = torch.randn(1000, C, device="cuda")
    dx = dres.clone()
    dg = torch.empty(C, device="cuda")
    db = torch.empty(C, device="cuda")
    ops.layernorm_bwd(x, dy, mu, rs, g, dx, dx, dg, db)
    yr.backward(dy.float())
    assert rel(dx - dres, xr.grad) <= 1e-4
    assert rel(dg, gr.grad) <= 1e-4
    assert rel(db, brr.grad) <= 1e-4


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("C,H,swap", [(128, 8, 0), (128, 8, 1), (32, 2, 0), (64, 4, 1), (16, 4, 0)])
def test_pair_bias_fwd_bwd_vs_torch(dtype, C, H, swap):
    from paper_2207_05477_b200 import ops
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    R = 48
    torch.manual_seed(C + H + swap)
    z = torch.randn(R * R, C, device="cuda").to(dt)
    g, b = torch.randn(C, device="cuda"), torch.randn(C, device="cuda") * 0.1
    w = torch.randn(C, H, device="cuda") * 0.2
    nb, mu, rs = ops.pair_bias_fwd(z, g, b, w, R, H, swap)
    zr = z.float().requires_grad_(True)
    gr, br_, wr = (t.clone().requires_grad_(True) for t in (g, b, w))
    P = torch.nn.functional.layer_norm(zr, (C,), gr, br_, 1e-5) @ wr      # [R*R, H]
    ref = P.view(R, R, H).permute(2, 0, 1)
    if swap:
        ref = ref.transpose(1, 2)
    tol = 1e-5 if dtype == "f32" else 1e-2
    assert rel(nb.float(), ref) <= tol
    dnb = torch.randn(H, R, R, device="cuda")
    dz0 = torch.randn(R * R, C, device="cuda")
    dz = dz0.clone()
    dg, db, dw = (torch.empty(C, device="cuda"), torch.empty(C, device="cuda"),
                  torch.empty(C, H, device="cuda"))
    ops.pair_bias_bwd(z, mu, rs, g, b, w, dnb, swap, dz, dg, db, dw, R, H)
    ref.backward(dnb)
    assert rel(dz - dz0, zr.grad) <= 1e-4
    assert rel(dg, gr.grad) <= 1e-4
    assert rel(db, br_.grad) <= 1e-4
    assert rel(dw, wr.grad) <= 1e-4


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("C", [64, 128, 256, 512, 1024, 96])
def test_colsum_relu_bias_kernels_vs_torch(dtype, C):
    from paper_2207_05477_b200 import ops
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    torch.manual_seed(C)
    rows = 3001
    x = torch.randn(rows, C, device="cuda")
    out = torch.empty(C, device="cuda")
    y = torch.empty(rows, C, device="cuda", dtype=dt)
    ops.colsum_cast(x, out, y=y)
    assert rel(out, x.double().sum(0).float()) <= 1e-5
    assert rel(y.float(), x.to(dt).float()) == 0.0
    h = torch.randn(rows, C, device="cuda").to(dt)
    dh = torch.randn(rows, C, device="cuda").to(dt)
    want = (dh.float() * (h.float() > 0))
    db = torch.empty(C, device="cuda")
    ops.relu_bwd_colsum_(dh, h, db)
    assert rel(dh.float(), want) == 0.0
    assert rel(db, want.sum(0)) <= 1e-5
    bias = torch.randn(C, device="cuda")
    res = torch.randn(rows, C, device="cuda").to(dt)
    yy = torch.randn(rows, C, device="cuda").to(dt)
    o = torch.empty_like(res)
    ops.bias_residual(res, yy, bias, o)
    assert rel(o.float(), (res.float() + (yy.float() + bias)).to(dt).float()) <= 1e-2 if dt == torch.bfloat16 else 1e-6


def test_layernorm_bwd_ex_fused_outputs():
    from paper_2207_05477_b200 import _lib, ops
    C, rows = 256, 4099
    x = torch.randn(rows, C, device="cuda").to(torch.bfloat16)
    g, b = torch.randn(C, device="cuda"), torch.randn(C, device="cuda")
    y, mu, rs = ops.layernorm(x, g, b, torch.bfloat16)
    dy = torch.randn(rows, C, device="cuda")
    dres = torch.randn(rows, C, device="cuda")
    dx = dres.clone()
    dx16 = torch.empty(rows, C, device="cuda", dtype=torch.bfloat16)
    dxs, dg, db = (torch.empty(C, device="cuda") for _ in range(3))
    ws = torch.empty(_lib.load().evo_layernorm_bwd_workspace(rows, C), dtype=torch.uint8, device="cuda")
    ops.call("evo_layernorm_bwd_ex", ops.ptr(x), ops.dcode(x), ops.ptr(dy), ops.dcode(dy), ops.ptr(mu),
             ops.ptr(rs), ops.ptr(g), ops.ptr(dx), ops.ptr(dx), ops.ptr(dx16), ops.ptr(dxs), ops.ptr(dg),
             ops.ptr(db), 0, ops.ptr(ws), rows, C, ops.stream())
    dx2 = dres.clone()
    dg2, db2 = torch.empty(C, device="cuda"), torch.empty(C, device="cuda")
    ops.layernorm_bwd(x, dy, mu, rs, g, dx2, dx2, dg2, db2)
    assert torch.equal(dx, dx2) and torch.equal(dg, dg2) and torch.equal(db, db2)
    assert torch.equal(dx16, dx.to(torch.bfloat16))
    assert rel(dxs, dx.double().sum(0).float()) <= 1e-5


@pytest.mark.parametrize("relu,with_res", [(False, True), (False, False), (True, False)])
@pytest.mark.parametrize("T,K,N", [(32768, 256, 256), (65536, 128, 512), (8192, 1024, 128)])
def test_gemm_bias_fused_epilogue_vs_torch(relu, with_res, T, K, N):
    """Projection + module epilogue (bias [+ residual] or bias + ReLU) in one
    kernel (evo_gemm_bias, tcgen05 GEMM epilogue) against fp32 torch, at the
    bench shapes where the fused path is taken."""
    from paper_2207_05477_b200 import ops
    torch.manual_seed(T + K + N)
    a = (torch.randn(T, K, device="cuda") * 0.5).bfloat16()
    w = (torch.randn(K, N, device="cuda") / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda") * 0.1
    res = torch.randn(T, N, device="cuda").bfloat16() if with_res else None
    out = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm_bias(a, w, out, bias, res=res, relu=relu)
    ref = a.float() @ w.float() + bias
    if with_res:
        ref = ref + res.float()
    if relu:
        ref = ref.clamp_min(0)
    assert rel(out.float(), ref) <= 1e-2


@pytest.mark.parametrize("geom", ["row", "col", "tri_start", "tri_end"])
def test_attention_bench_geometry_padded_mask(geom):
    """The bench geometries (N_seq=128, N_res=256, 8 heads): ~10-30 batches per
    CTA, and the bench features' padded residues, which make whole batches
    fully masked (column / triangle attention).  The bf16 tcgen05 path must stay
    finite and agree with the fp32 path on the same inputs -- this is the
    configuration where a cross-thread staging race once produced inf/NaN."""
    from paper_2207_05477_b200 import ops
    S, R, H = 128, 256, 8
    B, L, sb, sl, msb, msl = GEOMS[geom](S, R)
    C = 256 if geom in ("row", "col") else 128
    D = C // H
    T = S * R if geom in ("row", "col") else R * R
    torch.manual_seed(11)
    q32 = torch.randn(T, 4 * C, device="cuda") * 0.5
    mask = torch.ones(T, device="cuda")
    nv = R - R // 10
    mv = mask.view(S, R) if geom in ("row", "col") else mask.view(R, R)
    mv[:, nv:] = 0.0
    if geom in ("tri_start", "tri_end"):
        mv[nv:, :] = 0.0
    bias32 = torch.randn(H, L, L, device="cuda") * 0.1 if geom != "col" else None
    bg = torch.randn(C, device="cuda") * 0.1
    dg32 = torch.randn(T, C, device="cuda")
    out = {}
    for dt in (torch.float32, torch.bfloat16):
        q = q32.to(dt)
        bias = bias32.to(dt) if bias32 is not None else None
        ctx, gate, gated, lse = ops.attn_fwd(q, mask, msb, msl, bias, bg, B, L, H, D, sb, sl)
        dbg = torch.empty(C, device="cuda")
        dq, dnb = ops.attn_bwd(q, mask, msb, msl, bias, ctx, gate, dg32.to(dt), lse, dbg, B, L, H, D, sb, sl,
                               want_dbias=bias is not None)
        out[dt] = (ctx.float(), dq.float(), dnb)
    c32, d32, n32 = out[torch.float32]
    c16, d16, n16 = out[torch.bfloat16]
    assert torch.isfinite(c16).all() and torch.isfinite(d16).all()
    assert rel(c16, c32) <= 2e-2
    assert rel(d16, d32) <= 3e-2
    if n32 is not None:
        assert torch.isfinite(n16).all()
        assert rel(n16, n32) <= 3e-2


@pytest.mark.parametrize("name,S,R,H,D,geom", [("F_row", 512, 384, 8, 32, "row"), ("F_col", 512, 384, 8, 32, "col"),
                                                ("F_tri_end", 8, 384, 8, 16, "tri_end"),
                                                ("X_tri", 8, 1024, 4, 32, "tri_start")])
@pytest.mark.timeout(600)
def test_attention_long_rows_vs_fp32(name, S, R, H, D, geom):
    """L > 256 (fine-tune shape F, stress shape X): the key-blocked tcgen05
    forward against the fp32 path on the same inputs (padded masks, fully-masked
    batches included); for F also the backward (bf16 SIMT, fused logit order)."""
    from paper_2207_05477_b200 import ops
    B, L, sb, sl, msb, msl = GEOMS[geom](S, R)
    T = S * R if geom in ("row", "col") else R * R
    torch.manual_seed(5)
    q32 = torch.randn(T, 4 * H * D, device="cuda") * 0.5
    mask = torch.ones(T, device="cuda")
    nv = R - R // 10
    mv = mask.view(S, R) if geom in ("row", "col") else mask.view(R, R)
    mv[:, nv:] = 0.0
    if geom.startswith("tri"):
        mv[nv:, :] = 0.0
        mv[:3, :] = 0.0  # more fully-masked rows / masked keys
    bias32 = torch.randn(H, L, L, device="cuda") * 0.1 if geom != "col" else None
    bg = torch.randn(H * D, device="cuda") * 0.1
    dg32 = torch.randn(T, H * D, device="cuda")
    out = {}
    for dt in (torch.float32, torch.bfloat16):
        q = q32.to(dt)
        bias = bias32.to(dt) if bias32 is not None else None
        ctx, gate, gated, lse = ops.attn_fwd(q, mask, msb, msl, bias, bg, B, L, H, D, sb, sl)
        dq = None
        if name.startswith("F"):
            dbg = torch.empty(H * D, device="cuda")
            dq, _ = ops.attn_bwd(q, mask, msb, msl, bias, ctx, gate, dg32.to(dt), lse, dbg, B, L, H, D, sb, sl,
                                 want_dbias=bias is not None)
            dq = dq.float()
        out[dt] = (ctx.float(), dq)
    c32, d32 = out[torch.float32]
    c16, d16 = out[torch.bfloat16]
    assert torch.isfinite(c16).all()
    assert rel(c16, c32) <= 2e-2
    if d16 is not None:
        assert torch.isfinite(d16).all()
        assert rel(d16, d32) <= 3e-2


@pytest.mark.parametrize("C", [128, 256])
@pytest.mark.parametrize("rows,dy_dt,with_res", [(8192, "f32", True), (8196, "f32", False),
                                                 (65536, "bf16", True), (4100, "f32", True)])
def test_layernorm_bwd_stream_vs_torch(C, rows, dy_dt, with_res):
    """The bulk-copy-staged LayerNorm backward (csrc/glue_stream.cu; taken for
    bf16 x, rows % 4 == 0, rows >= 4096) against fp32 torch, including a
    partial last stage (8196 rows) and the fused bf16 copy / column sums."""
    from paper_2207_05477_b200 import _lib, ops
    torch.manual_seed(rows + C)
    x = (torch.randn(rows, C, device="cuda") * 2 + 0.5).bfloat16()
    g, b = torch.randn(C, device="cuda"), torch.randn(C, device="cuda")
    y, mu, rs = ops.layernorm(x, g, b, torch.bfloat16)
    dy = torch.randn(rows, C, device="cuda").to(torch.float32 if dy_dt == "f32" else torch.bfloat16)
    dres = torch.randn(rows, C, device="cuda") if with_res else None
    dx = dres.clone() if with_res else torch.empty(rows, C, device="cuda")
    dg, db = torch.empty(C, device="cuda"), torch.empty(C, device="cuda")
    ops.layernorm_bwd(x, dy, mu, rs, g, dx if with_res else None, dx, dg, db)
    xr = x.float().requires_grad_(True)
    gr, br_ = g.clone().requires_grad_(True), b.clone().requires_grad_(True)
    torch.nn.functional.layer_norm(xr, (C,), gr, br_, 1e-5).backward(dy.float())
    got = dx - dres if with_res else dx
    assert rel(got, xr.grad) <= 1e-4
    assert rel(dg, gr.grad) <= 1e-4 and rel(db, br_.grad) <= 1e-4
    # fused outputs: bf16 copy of dx and its column sums
    dx2 = dres.clone() if with_res else torch.zeros(rows, C, device="cuda")
    dx16 = torch.empty(rows, C, device="cuda", dtype=torch.bfloat16)
    dxs, dg2, db2 = (torch.empty(C, device="cuda") for _ in range(3))
    ws = torch.empty(_lib.load().evo_layernorm_bwd_workspace(rows, C), dtype=torch.uint8, device="cuda")
    ops.call("evo_layernorm_bwd_ex", ops.ptr(x), ops.dcode(x), ops.ptr(dy), ops.dcode(dy), ops.ptr(mu),
             ops.ptr(rs), ops.ptr(g), ops.ptr(dx2), ops.ptr(dx2), ops.ptr(dx16), ops.ptr(dxs), ops.ptr(dg2),
             ops.ptr(db2), 0, ops.ptr(ws), rows, C, ops.stream())
    assert torch.equal(dx16, dx2.to(torch.bfloat16))
    assert rel(dxs, dx2.double().sum(0).float()) <= 1e-5
    assert rel(dx2 - (dres if with_res else 0), xr.grad) <= 1e-4


@pytest.mark.parametrize("NI,NJ,swap", [(256, 256, 0), (256, 256, 1), (128, 256, 0), (256, 128, 1),
                                        (100, 82, 0)])
def test_pair_bias_bwd_stream_vs_torch(NI, NJ, swap):
    """The bulk-copy-staged pair-bias backward (csrc/glue_stream.cu; bf16,
    C = 128, >= 4096 tokens) against fp32 torch, square and rectangular (DAP
    shard) extents, both bias layouts, and a partial last stage (100 x 82)."""
    from paper_2207_05477_b200 import ops
    C, H = 128, 8
    torch.manual_seed(NI + NJ + swap)
    z = torch.randn(NI * NJ, C, device="cuda").bfloat16()
    g, b = torch.randn(C, device="cuda"), torch.randn(C, device="cuda") * 0.1
    w = torch.randn(C, H, device="cuda") * 0.2
    nb, mu, rs = ops.pair_bias_fwd(z, g, b, w, 0, H, swap, ni=NI, nj=NJ)
    zr = z.float().requires_grad_(True)
    gr, br_, wr = (t.clone().requires_grad_(True) for t in (g, b, w))
    P = torch.nn.functional.layer_norm(zr, (C,), gr, br_, 1e-5) @ wr
    ref = P.view(NI, NJ, H).permute(2, 0, 1)
    if swap:
        ref = ref.transpose(1, 2)
    assert rel(nb.float(), ref) <= 1e-2
    dnb = torch.randn(ref.shape, device="cuda").contiguous()
    dz0 = torch.randn(NI * NJ, C, device="cuda")
    dz = dz0.clone()
    dg, db, dw = torch.empty(C, device="cuda"), torch.empty(C, device="cuda"), torch.empty(C, H, device="cuda")
    ops.pair_bias_bwd(z, mu, rs, g, b, w, dnb, swap, dz, dg, db, dw, 0, H, ni=NI, nj=NJ)
    ref.backward(dnb)
    assert rel(dz - dz0, zr.grad) <= 1e-4
    assert rel(dg, gr.grad) <= 1e-4 and rel(db, br_.grad) <= 1e-4 and rel(dw, wr.grad) <= 1e-4


@pytest.mark.parametrize("C", [128, 256])
@pytest.mark.parametrize("rows,ydt", [(8192, "bf16"), (8200, "bf16"), (65536, "f32")])
def test_layernorm_fwd_stream_vs_torch(C, rows, ydt):
    """Bulk-copy-staged LayerNorm forward (bf16 x, >= 4096 rows) against fp32
    torch, including a partial last stage."""
    from paper_2207_05477_b200 import ops
    torch.manual_seed(rows + C)
    x = (torch.randn(rows, C, device="cuda") * 2 + 0.5).bfloat16()
    g, b = torch.randn(C, device="cuda"), torch.randn(C, device="cuda")
    dt = torch.bfloat16 if ydt == "bf16" else torch.float32
    y, mu, rs = ops.layernorm(x, g, b, dt)
    ref = torch.nn.functional.layer_norm(x.float(), (C,), g, b, 1e-5)
    assert rel(y.float(), ref) <= (1e-2 if ydt == "bf16" else 1e-5)
    xf = x.float()
    assert rel(mu, xf.mean(1)) <= 1e-5
    assert rel(rs, torch.rsqrt(xf.var(1, unbiased=False) + 1e-5)) <= 1e-4


@pytest.mark.parametrize("R,ni", [(256, 256), (256, 128), (384, 384)])
def test_opm_dnum_tc_vs_torch(R, ni):
    """OPM backward d(pair) -> d(num) as one tcgen05 GEMM with the normalisation
    and [i*k+p, j*k+q] re-layout in the epilogue (csrc/opm_tc.cu), against
    fp32 torch; ni < R is a DAP row shard."""
    from paper_2207_05477_b200 import ops
    k, C = 32, 128
    torch.manual_seed(R + ni)
    d_act = (torch.randn(ni * R, C, device="cuda") * 0.5).bfloat16()
    w_out = (torch.randn(k * k, C, device="cuda") * 0.1).bfloat16()
    rec = torch.rand(ni * R, device="cuda") + 0.01
    dnum = ops.opm_dnum(d_act, w_out, rec, R, k, ni=ni)
    assert dnum is not None and dnum.shape == (ni * k, R * k)
    doutn = (d_act.float() @ w_out.float().t()) * rec[:, None]          # [(i, j), (p, q)]
    ref = doutn.view(ni, R, k, k).permute(0, 2, 1, 3).reshape(ni * k, R * k)
    assert rel(dnum.float(), ref) <= 1e-2


@pytest.mark.parametrize("R", [256, 384])
def test_opm_outn_tc_vs_torch(R):
    """OPM forward: sum over sequences + normalisation + [(i, j), p*k+q]
    re-layout as one tcgen05 GEMM (csrc/opm_tc.cu) against fp32 torch."""
    from paper_2207_05477_b200 import ops
    S, k = 128, 32
    torch.manual_seed(R)
    a = (torch.randn(S, R * k, device="cuda") * 0.3).bfloat16()
    c = (torch.randn(S, R * k, device="cuda") * 0.3).bfloat16()
    rec = torch.rand(R * R, device="cuda") + 0.01
    outn = ops.opm_outn(a, c, rec, S, R, k)
    assert outn is not None and outn.shape == (R * R, k * k)
    num = a.float().t() @ c.float()                                      # [(i, p), (j, q)]
    ref = num.view(R, k, R, k).permute(0, 2, 1, 3).reshape(R * R, k * k) * rec[:, None]
    assert rel(outn.float(), ref) <= 1e-2


@pytest.mark.parametrize("A,B,E,dt", [(8, 4, 256, torch.bfloat16), (3, 5, 7, torch.bfloat16), (16, 2, 33, torch.float32)])
def test_swap01_vs_torch(A, B, E, dt):
    """DAP outer-axis swap (csrc/dap.cu): dst[b, a, :] = src[a, b, :] for 16-B,
    4-B and byte-granular row sizes."""
    from paper_2207_05477_b200 import ops
    x = torch.randn(A, B, E, device="cuda").to(dt)
    y = ops.swap01(x, A, B)
    assert torch.equal(y.view(B, A, E), x.permute(1, 0, 2))


def test_opm_rec_once_per_pass_matches_inline():
    """The normaliser computed once (evo_opm_rec) and applied per block
    (evo_opm_norm_apply_rows) equals the inline evo_opm_norm_fwd_rows, full and
    for a row shard."""
    from paper_2207_05477_b200 import ops
    S, R, k = 24, 64, 32
    torch.manual_seed(5)
    mask = (torch.rand(S * R, device="cuda") > 0.2).float()
    num = torch.randn(R * k, R * k, device="cuda").bfloat16()
    rec0, out0 = ops.opm_norm_fwd(num, mask, S, R, k, torch.bfloat16)
    rec = ops.opm_rec(mask, S, R)
    _, out1 = ops.opm_norm_fwd(num, mask, S, R, k, torch.bfloat16, rec=rec)
    assert torch.equal(rec0, rec) and torch.equal(out0, out1)
    rec_s = ops.opm_rec(mask, S, R, i0=16, ni=32)
    assert torch.equal(rec_s, rec.view(R, R)[16:48].reshape(-1))


@pytest.mark.parametrize("NI,NJ,swap", [(256, 256, 0), (256, 256, 1), (128, 256, 0), (256, 128, 1),
                                        (100, 82, 0), (82, 100, 1)])
def test_ln_pair_bias_fused_vs_torch(NI, NJ, swap):
    """Triangle attention's input LayerNorm and its pair bias in one pass
    (csrc/pair_bias_mma.cu, LN = true) against fp32 torch: xl and nb within
    bf16 rounding, the shared row statistics to fp32 accuracy; the unfused
    ops agree with it."""
    from paper_2207_05477_b200 import ops
    C, H = 128, 8
    torch.manual_seed(NI * 3 + NJ + swap)
    z = (torch.randn(NI * NJ, C, device="cuda") * 1.5 + 0.3).bfloat16()
    lg, lb = torch.randn(C, device="cuda"), torch.randn(C, device="cuda") * 0.1
    g, b = torch.randn(C, device="cuda"), torch.randn(C, device="cuda") * 0.1
    w = torch.randn(C, H, device="cuda") * 0.2
    out = ops.ln_pair_bias_fwd(z, lg, lb, g, b, w, 0, H, swap, ni=NI, nj=NJ)
    assert out is not None
    xl, nb, mu, rs = out
    zf = z.float()
    assert rel(xl.float(), torch.nn.functional.layer_norm(zf, (C,), lg, lb, 1e-5)) <= 1e-2
    P = torch.nn.functional.layer_norm(zf, (C,), g, b, 1e-5) @ w
    ref = P.view(NI, NJ, H).permute(2, 0, 1)
    if swap:
        ref = ref.transpose(1, 2)
    assert rel(nb.float(), ref) <= 1e-2
    assert rel(mu, zf.mean(1)) <= 1e-5
    assert rel(rs, torch.rsqrt(zf.var(1, unbiased=False) + 1e-5)) <= 1e-5
    nb2, mu2, rs2 = ops.pair_bias_fwd(z, g, b, w, 0, H, swap, ni=NI, nj=NJ)
    xl2, _, _ = ops.layernorm(z, lg, lb, torch.bfloat16)
    assert rel(nb.float(), nb2.float()) <= 1e-2 and rel(xl.float(), xl2.float()) <= 1e-2


@pytest.mark.parametrize("swap", [0, 1])
def test_pair_bias_bwd_emits_next_operand(swap):
    """pair_bias_bwd with dz16 / dzsum (the last write to the pair gradient):
    the same dz, dgamma, dbeta, dw as without, plus bf16(dz) and its column
    sums in the same pass (csrc/glue_stream.cu)."""
    from paper_2207_05477_b200 import ops
    R, C, H = 256, 128, 8
    torch.manual_seed(17 + swap)
    z = torch.randn(R * R, C, device="cuda").bfloat16()
    g, b = torch.randn(C, device="cuda"), torch.randn(C, device="cuda") * 0.1
    w = torch.randn(C, H, device="cuda") * 0.2
    _, mu, rs = ops.pair_bias_fwd(z, g, b, w, R, H, swap)
    dnb = torch.randn(H, R, R, device="cuda")
    dz0 = torch.randn(R * R, C, device="cuda")
    outs = []
    for fused in (False, True):
        dz = dz0.clone()
        dg, db, dw = torch.empty(C, device="cuda"), torch.empty(C, device="cuda"), torch.empty(C, H, device="cuda")
        d16 = torch.empty(R * R, C, device="cuda", dtype=torch.bfloat16) if fused else None
        dsum = torch.full((C,), 3.0, device="cuda") if fused else None
        ops.pair_bias_bwd(z, mu, rs, g, b, w, dnb, swap, dz, dg, db, dw, R, H, dz16=d16, dzsum=dsum)
        outs.append((dz, dg, db, dw, d16, dsum))
    (dz, dg, db, dw, _, _), (dzf, dgf, dbf, dwf, d16, dsum) = outs
    assert torch.equal(dz, dzf) and torch.equal(dg, dgf) and torch.equal(db, dbf) and torch.equal(dw, dwf)
    assert torch.equal(d16, dzf.bfloat16())
    assert rel(dsum, dzf.double().sum(0).float()) <= 1e-5


@pytest.mark.parametrize("rows,cols,src", [(128, 4096, "bf16"), (4096, 128, "f32"), (96, 200, "bf16")])
def test_transpose2d_vs_torch(rows, cols, src):
    """evo_transpose2d (TriMul's channel-major <-> token-major re-layouts): the
    16-byte tiled kernel (multiples of 64) and the scalar one, exact."""
    from paper_2207_05477_b200 import ops
    torch.manual_seed(rows + cols)
    x = torch.randn(rows, cols, device="cuda")
    if src == "bf16":
        x = x.bfloat16()
    y = ops.transpose2d(x, torch.bfloat16)
    assert torch.equal(y, x.t().contiguous().bfloat16())
