"""Numpy restatement of the reference Evoformer hot path (CPU oracle).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  This module is the
checker for the sm_100a kernels, never the thing measured or shipped.

Every function follows the reference package ``evotrain``
(``/root/reference/pkg/src/evotrain``, abbreviated ``src/``) and cites the
file:line it restates.  Arithmetic is float32 throughout, with the same op
order as the reference where that order is observable at fp32 (mask/bias
accumulation into the logits, ``recip`` then multiply in the OPM, ...).
Backward passes are written out per module (the reference gets them from
its tape, ``src/autodiff.py:84-99``, whose per-op closures live in
``src/tensor.py:133-435`` and ``src/attention.py:178-221``).

Parity of this restatement against the reference itself is pinned by
``tests/test_oracle_golden.py`` (goldens made by ``tests/golden/gen_goldens.py``
from the reference).  ``trimul_*`` has NO reference counterpart (the
reference lists TriangleMultiplication only as planner inventory,
``src/planner.py:37-45``); it restates AlphaFold2 Supplementary Algorithms
11/12 and its parity is UNPINNED.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

F32 = np.float32

# ---------------------------------------------------------------------------
# PRNG: splitmix64, vectorised (src/prng.py:19-53).  The reference steps a
# Python int per draw; state_i = seed + i*GAMMA (mod 2^64), so the stream is
# computable in one numpy pass with identical bits.

MASK64 = (1 << 64) - 1
GAMMA = np.uint64(0x9E3779B97F4A7C15)
MIX1 = np.uint64(0xBF58476D1CE4E5B9)
MIX2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * MIX1
        z = (z ^ (z >> np.uint64(27))) * MIX2
    return z ^ (z >> np.uint64(31))


def splitmix64(seed: int, n: int = 1) -> list:
    """src/prng.py:19-31."""
    return [int(v) for v in _stream(seed & MASK64, 0, n)]


def _stream(state: int, start: int, n: int) -> np.ndarray:
    i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        s = np.uint64(state) + i * GAMMA
    return _mix(s)


class Prng:
    """src/prng.py:34-53 (``next_u64`` / ``uniform``), vectorised."""

    def __init__(self, seed: int):
        self._seed = seed & MASK64
        self._count = 0

    def uniform(self, shape, low: float = -1.0, high: float = 1.0) -> np.ndarray:
        n = int(np.prod(shape)) if shape else 1
        z = _stream(self._seed, self._count, n)
        self._count += n
        u = (z >> np.uint64(40)).astype(np.float64) / float(1 << 24)
        return (low + (high - low) * u).astype(F32).reshape(shape)


# ---------------------------------------------------------------------------
# configuration (src/model.py:42-65)


@dataclass
class ModelConfig:
    n_blocks: int = 2
    n_seq: int = 8
    n_res: int = 8
    c_m: int = 8
    c_z: int = 8
    heads: int = 2
    opm_dim: int = 4
    transition_factor: int = 4
    feat_dim: int = 8
    pad_fraction: float = 0.1
    # extension (absent from the reference, default off for parity):
    # TriangleMultiplication outgoing+incoming inserted after ``pair += opm``.
    trimul: bool = False
    trimul_hidden: int = 0  # 0 -> c_z

    @property
    def c_hidden_mul(self) -> int:
        return self.trimul_hidden or self.c_z


ATTN_FIELDS = ("wq", "wk", "wv", "wg", "bg", "wo", "bo")
MSA_BRANCH_MODULES = ("row_attn", "col_attn", "msa_trans", "opm")
PAIR_BRANCH_MODULES = ("tri_start", "tri_end", "pair_trans")
TRIMUL_MODULES = ("tri_mul_out", "tri_mul_in")
TRIMUL_SEED_SALT = 0x5EED7A1


def param_specs(cfg: ModelConfig):
    """(name, shape, kind) in the reference flatten order
    (src/model.py:203-220); kind is 'u' (uniform*0.1), 'ones' or 'zeros'
    exactly as ``init_params`` draws them (src/model.py:140-200)."""
    H = cfg.heads
    specs = [
        ("msa_embed.w", (cfg.feat_dim, cfg.c_m), "u"), ("msa_embed.b", (cfg.c_m,), "zeros"),
        ("pair_embed.w", (cfg.feat_dim, cfg.c_z), "u"), ("pair_embed.b", (cfg.c_z,), "zeros"),
        ("recycle_m.g", (cfg.c_m,), "ones"), ("recycle_m.b", (cfg.c_m,), "zeros"),
        ("recycle_z.g", (cfg.c_z,), "ones"), ("recycle_z.b", (cfg.c_z,), "zeros"),
    ]

    def attn(prefix, c, bias_from):
        hd = c // H
        out = [(f"{prefix}.ln_g", (c,), "ones"), (f"{prefix}.ln_b", (c,), "zeros")]
        for f in ("wq", "wk", "wv", "wg"):
            out.append((f"{prefix}.attn.{f}", (c, H, hd), "u"))
        out += [(f"{prefix}.attn.bg", (H, hd), "zeros"),
                (f"{prefix}.attn.wo", (H, hd, c), "u"),
                (f"{prefix}.attn.bo", (c,), "zeros")]
        if bias_from:
            out += [(f"{prefix}.bias_ln_g", (bias_from,), "ones"),
                    (f"{prefix}.bias_ln_b", (bias_from,), "zeros"),
                    (f"{prefix}.w_bias", (bias_from, H), "u")]
        return out

    def trans(prefix, c):
        f = cfg.transition_factor
        return [(f"{prefix}.ln_g", (c,), "ones"), (f"{prefix}.ln_b", (c,), "zeros"),
                (f"{prefix}.w1", (c, f * c), "u"), (f"{prefix}.b1", (f * c,), "zeros"),
                (f"{prefix}.w2", (f * c, c), "u"), (f"{prefix}.b2", (c,), "zeros")]

    for i in range(cfg.n_blocks):
        p = f"block{i}"
        k = cfg.opm_dim
        specs += attn(f"{p}.row_attn", cfg.c_m, cfg.c_z)
        specs += attn(f"{p}.col_attn", cfg.c_m, 0)
        specs += trans(f"{p}.msa_trans", cfg.c_m)
        specs += [(f"{p}.opm.ln_g", (cfg.c_m,), "ones"), (f"{p}.opm.ln_b", (cfg.c_m,), "zeros"),
                  (f"{p}.opm.w_left", (cfg.c_m, k), "u"), (f"{p}.opm.b_left", (k,), "zeros"),
                  (f"{p}.opm.w_right", (cfg.c_m, k), "u"), (f"{p}.opm.b_right", (k,), "zeros"),
                  (f"{p}.opm.w_out", (k * k, cfg.c_z), "u"), (f"{p}.opm.b_out", (cfg.c_z,), "zeros")]
        specs += attn(f"{p}.tri_start", cfg.c_z, cfg.c_z)
        specs += attn(f"{p}.tri_end", cfg.c_z, cfg.c_z)
        specs += trans(f"{p}.pair_trans", cfg.c_z)
        if cfg.trimul:
            for m in TRIMUL_MODULES:
                specs += trimul_specs(f"{p}.{m}", cfg.c_z, cfg.c_hidden_mul)
    return specs


def trimul_specs(prefix, cz, ch):
    """Extension parameter set (AF2 Alg 11/12)."""
    return [(f"{prefix}.ln_in_g", (cz,), "ones"), (f"{prefix}.ln_in_b", (cz,), "zeros"),
            (f"{prefix}.w_ap", (cz, ch), "tu"), (f"{prefix}.b_ap", (ch,), "zeros"),
            (f"{prefix}.w_ag", (cz, ch), "tu"), (f"{prefix}.b_ag", (ch,), "zeros"),
            (f"{prefix}.w_bp", (cz, ch), "tu"), (f"{prefix}.b_bp", (ch,), "zeros"),
            (f"{prefix}.w_bg", (cz, ch), "tu"), (f"{prefix}.b_bg", (ch,), "zeros"),
            (f"{prefix}.ln_out_g", (ch,), "ones"), (f"{prefix}.ln_out_b", (ch,), "zeros"),
            (f"{prefix}.w_o", (ch, cz), "tu"), (f"{prefix}.b_o", (cz,), "zeros"),
            (f"{prefix}.w_g", (cz, cz), "tu"), (f"{prefix}.b_g", (cz,), "zeros")]


def init_params(cfg: ModelConfig, seed: int) -> dict:
    """src/model.py:172-200: uniform[-1,1)*0.1 weights in draw order, ones
    for LN gains, zeros for biases.  TriMul weights ('tu') come from a
    separate stream so the reference parameters stay bit-identical."""
    rng = Prng(seed)
    trng = Prng(seed ^ TRIMUL_SEED_SALT)
    out = {}
    for name, shape, kind in param_specs(cfg):
        if kind == "u":
            out[name] = rng.uniform(shape) * F32(0.1)
        elif kind == "tu":
            out[name] = trng.uniform(shape) * F32(0.1)
        elif kind == "ones":
            out[name] = np.ones(shape, F32)
        else:
            out[name] = np.zeros(shape, F32)
    return out


def branch_param_names(cfg: ModelConfig, branch: str) -> set:
    """src/model.py:223-236 (TriMul joins the pair branch)."""
    embeds = {"msa": ("msa_embed.", "recycle_m."), "pair": ("pair_embed.", "recycle_z.")}[branch]
    mods = MSA_BRANCH_MODULES if branch == "msa" else PAIR_BRANCH_MODULES + TRIMUL_MODULES
    names = set()
    for name, _, _ in param_specs(cfg):
        if name.startswith(embeds):
            names.add(name)
        elif name.startswith("block") and name.split(".")[1] in mods:
            names.add(name)
    return names


@dataclass
class Features:
    msa_feat: np.ndarray
    pair_feat: np.ndarray
    msa_mask: np.ndarray
    pair_mask: np.ndarray


def make_features(cfg: ModelConfig, seed: int) -> Features:
    """src/model.py:274-288."""
    rng = Prng(seed)
    s, r, f = cfg.n_seq, cfg.n_res, cfg.feat_dim
    n_valid = r - int(np.floor(cfg.pad_fraction * r))
    msa_mask = np.ones((1, s, r), F32)
    msa_mask[:, :, n_valid:] = 0.0
    pair_mask = np.ones((1, r, r), F32)
    pair_mask[:, n_valid:, :] = 0.0
    pair_mask[:, :, n_valid:] = 0.0
    msa_feat = rng.uniform((1, s, r, f))
    pair_feat = rng.uniform((1, r, r, f))
    return Features(msa_feat, pair_feat, msa_mask, pair_mask)


def draw_num_recycles(base_seed: int, step: int) -> int:
    """src/model.py:291-293."""
    return 1 + int(splitmix64(base_seed + step, 1)[0] % 4)


def step_feature_seed(base_seed: int, step: int) -> int:
    """src/trainer.py:98-101."""
    return int(splitmix64(base_seed + step, 2)[1] & 0x7FFFFFFF)


# ---------------------------------------------------------------------------
# primitives (src/tensor.py)


def bf16_round(arr: np.ndarray) -> np.ndarray:
    """src/tensor.py:37-43 (RNE onto the top 16 bits)."""
    u = np.ascontiguousarray(arr, dtype=F32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.view(F32).reshape(arr.shape)


def _sumto(g: np.ndarray, n: int) -> np.ndarray:
    return g.reshape(-1, n).sum(axis=0).astype(F32)


def _wgrad(x: np.ndarray, g: np.ndarray) -> np.ndarray:
    """d(x @ W)/dW for x [..., K], g [..., N]."""
    return (x.reshape(-1, x.shape[-1]).T @ g.reshape(-1, g.shape[-1])).astype(F32)


def ln_fwd(x, g, b, eps=1e-5):
    """src/tensor.py:173-185."""
    mu = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    inv = F32(1.0) / np.sqrt(var + F32(eps))
    xhat = (x - mu) * inv
    return (xhat * g + b).astype(F32), (x, g, eps)


def ln_bwd(dout, cache):
    """src/tensor.py:187-206 (statistics recomputed from x, as there)."""
    x, g, eps = cache
    n = x.shape[-1]
    mu = x.mean(axis=-1, keepdims=True)
    inv = F32(1.0) / np.sqrt(x.var(axis=-1, keepdims=True) + F32(eps))
    xh = (x - mu) * inv
    dgamma = _sumto(dout * xh, n)
    dbeta = _sumto(dout, n)
    dxh = dout * g
    dx = inv * (dxh - dxh.mean(axis=-1, keepdims=True)
                - xh * (dxh * xh).mean(axis=-1, keepdims=True))
    return dx.astype(F32), dgamma, dbeta


def sigmoid(x):
    """src/tensor.py:290-292."""
    return (F32(1.0) / (F32(1.0) + np.exp(-x))).astype(F32)


# ---------------------------------------------------------------------------
# fused gated attention (src/attention.py:118-233)


def attention_fwd(x, mask, nb, p):
    """``gated_attention_fused`` forward, src/attention.py:121-174.

    x [B,S,R,C], mask [B,S,R] in {0,1}, nb [H,R,R] or None,
    p: dict with wq/wk/wv/wg [C,H,c], bg [H,c], wo [H,c,C], bo [C].
    """
    b, s, r, cdim = x.shape
    h, c = p["wq"].shape[1], p["wq"].shape[2]
    hc = h * c
    inv_sqrt_c = F32(1.0 / np.sqrt(c))
    wqkv = np.concatenate([p["wq"].reshape(cdim, hc), p["wk"].reshape(cdim, hc),
                           p["wv"].reshape(cdim, hc)], axis=1)
    qkv = np.matmul(x, wqkv)

    def heads(flat):
        return flat.reshape(b, s, r, h, c).transpose(0, 1, 3, 2, 4)

    q5, k5, v5 = heads(qkv[..., :hc]), heads(qkv[..., hc:2 * hc]), heads(qkv[..., 2 * hc:])
    maskbias = (mask - F32(1.0)) * F32(1e9)                      # :151
    logits = np.matmul(q5, k5.swapaxes(-1, -2)) * inv_sqrt_c     # :153
    logits += maskbias[:, :, None, None, :]                      # :154
    if nb is not None:
        logits += nb[None, None]                                 # :156
    if logits.dtype != np.float32:
        # float64 evaluation (serial_grads_f64): keep the fp32 mask-bias
        # semantics -- at -1e9 every logit of a fully-masked row rounds to the
        # same fp32 value, so the row is uniform
        logits = logits.astype(np.float32).astype(logits.dtype)
    m = logits.max(axis=-1, keepdims=True)                       # :159-161
    e = np.exp(logits - m)
    w = (e / e.sum(axis=-1, keepdims=True)).astype(F32)
    ctx5 = np.matmul(w, v5)
    ctxf = ctx5.transpose(0, 1, 3, 2, 4).reshape(b, s, r, hc)
    gate = sigmoid(np.matmul(x, p["wg"].reshape(cdim, hc)) + p["bg"].reshape(hc))
    out = (np.matmul(ctxf * gate, p["wo"].reshape(hc, cdim)) + p["bo"]).astype(F32)
    cache = dict(x=x, nb=nb, p=p, qkv=qkv, w=w, ctxf=ctxf, gate=gate, wqkv=wqkv,
                 dims=(b, s, r, cdim, h, c))
    return out, cache


def attention_bwd(g, cache):
    """``gated_attention_fused`` backward closure, src/attention.py:178-221.
    Returns (dx, dparams, dnb)."""
    b, s, r, cdim, h, c = cache["dims"]
    hc = h * c
    p, x, qkv, w, ctxf, gate = (cache[k] for k in ("p", "x", "qkv", "w", "ctxf", "gate"))
    inv_sqrt_c = F32(1.0 / np.sqrt(c))
    g = g.astype(F32)
    wo_flat = p["wo"].reshape(hc, cdim)
    gated = ctxf * gate
    dwo = _wgrad(gated, g)
    dbo = _sumto(g, cdim)
    dgated = np.matmul(g, wo_flat.T)
    dctxf = dgated * gate
    dgate = dgated * ctxf
    dgp = dgate * gate * (F32(1.0) - gate)
    dwg = _wgrad(x, dgp)
    dbg = _sumto(dgp, hc)
    dx = np.matmul(dgp, p["wg"].reshape(cdim, hc).T)

    def heads(flat):
        return flat.reshape(b, s, r, h, c).transpose(0, 1, 3, 2, 4)

    q5, k5, v5 = heads(qkv[..., :hc]), heads(qkv[..., hc:2 * hc]), heads(qkv[..., 2 * hc:])
    dctx5 = heads(dctxf)
    dw = np.matmul(dctx5, v5.swapaxes(-1, -2))
    dv5 = np.matmul(w.swapaxes(-1, -2), dctx5)
    dlogits = w * (dw - (dw * w).sum(axis=-1, keepdims=True))
    dq5 = np.matmul(dlogits, k5) * inv_sqrt_c
    dk5 = np.matmul(dlogits.swapaxes(-1, -2), q5) * inv_sqrt_c

    def flat(d5):
        return d5.transpose(0, 1, 3, 2, 4).reshape(b, s, r, hc)

    dqkv = np.concatenate([flat(dq5), flat(dk5), flat(dv5)], axis=-1)
    dx = (dx + np.matmul(dqkv, cache["wqkv"].T)).astype(F32)
    dwqkv = _wgrad(x, dqkv)
    dp = dict(wq=dwqkv[:, :hc].reshape(cdim, h, c), wk=dwqkv[:, hc:2 * hc].reshape(cdim, h, c),
              wv=dwqkv[:, 2 * hc:].reshape(cdim, h, c), wg=dwg.reshape(cdim, h, c),
              bg=dbg.reshape(h, c), wo=dwo.reshape(h, c, cdim), bo=dbo)
    dnb = dlogits.sum(axis=(0, 1)).astype(F32) if cache["nb"] is not None else None
    return dx, dp, dnb


# ---------------------------------------------------------------------------
# block modules (src/model.py:300-445)


def _attn_p(P, prefix):
    return {f: P[f"{prefix}.attn.{f}"] for f in ATTN_FIELDS}


def pair_bias_fwd(z, P, prefix):
    """``_pair_bias``, src/model.py:312-317: LN(z)·w_bias -> [H,R,R]."""
    zl, ln_c = ln_fwd(z, P[f"{prefix}.bias_ln_g"], P[f"{prefix}.bias_ln_b"])
    nb = np.matmul(zl, P[f"{prefix}.w_bias"])                    # [1,R,R,H]
    nb = np.ascontiguousarray(nb.reshape(nb.shape[1:]).transpose(2, 0, 1))
    return nb, (zl, ln_c)


def pair_bias_bwd(dnb, cache, P, prefix, grads):
    zl, ln_c = cache
    d = np.ascontiguousarray(dnb.transpose(1, 2, 0))[None]      # [1,R,R,H]
    _acc(grads, f"{prefix}.w_bias", _wgrad(zl, d))
    dz, dg, db = ln_bwd(np.matmul(d, P[f"{prefix}.w_bias"].T), ln_c)
    _acc(grads, f"{prefix}.bias_ln_g", dg)
    _acc(grads, f"{prefix}.bias_ln_b", db)
    return dz


def _acc(grads, name, g):
    g = np.asarray(g, F32)
    if name in grads:
        grads[name] = grads[name] + g
    else:
        grads[name] = g.copy()


def _acc_attn(grads, prefix, dp):
    for f in ATTN_FIELDS:
        _acc(grads, f"{prefix}.attn.{f}", dp[f])


def row_attn_fwd(msa, pair, msa_mask, P, prefix):
    """``msa_row_attention``, src/model.py:320-328."""
    x, ln_c = ln_fwd(msa, P[f"{prefix}.ln_g"], P[f"{prefix}.ln_b"])
    nb, nb_c = pair_bias_fwd(pair, P, prefix)
    y, a_c = attention_fwd(x, msa_mask, nb, _attn_p(P, prefix))
    return msa + y, (ln_c, nb_c, a_c)


def row_attn_bwd(dout, cache, P, prefix, grads):
    ln_c, nb_c, a_c = cache
    dx, dp, dnb = attention_bwd(dout, a_c)
    _acc_attn(grads, prefix, dp)
    dmsa, dg, db = ln_bwd(dx, ln_c)
    _acc(grads, f"{prefix}.ln_g", dg)
    _acc(grads, f"{prefix}.ln_b", db)
    dpair = pair_bias_bwd(dnb, nb_c, P, prefix, grads)
    return dout + dmsa, dpair


def col_attn_fwd(msa, msa_mask_t, P, prefix):
    """``msa_col_attention``, src/model.py:331-341 (serial: alltoall = id)."""
    xt = np.ascontiguousarray(msa.transpose(0, 2, 1, 3))
    x, ln_c = ln_fwd(xt, P[f"{prefix}.ln_g"], P[f"{prefix}.ln_b"])
    y, a_c = attention_fwd(x, msa_mask_t, None, _attn_p(P, prefix))
    return msa + np.ascontiguousarray(y.transpose(0, 2, 1, 3)), (ln_c, a_c)


def col_attn_bwd(dout, cache, P, prefix, grads):
    ln_c, a_c = cache
    dy = np.ascontiguousarray(dout.transpose(0, 2, 1, 3))
    dx, dp, _ = attention_bwd(dy, a_c)
    _acc_attn(grads, prefix, dp)
    dxt, dg, db = ln_bwd(dx, ln_c)
    _acc(grads, f"{prefix}.ln_g", dg)
    _acc(grads, f"{prefix}.ln_b", db)
    return dout + np.ascontiguousarray(dxt.transpose(0, 2, 1, 3))


def transition_fwd(x, P, prefix):
    """``transition``, src/model.py:344-348."""
    h, ln_c = ln_fwd(x, P[f"{prefix}.ln_g"], P[f"{prefix}.ln_b"])
    a = np.matmul(h, P[f"{prefix}.w1"]) + P[f"{prefix}.b1"]
    rl = np.maximum(a, F32(0.0))
    o = np.matmul(rl, P[f"{prefix}.w2"]) + P[f"{prefix}.b2"]
    return (x + o).astype(F32), (ln_c, h, rl)


def transition_bwd(dout, cache, P, prefix, grads):
    ln_c, h, rl = cache
    _acc(grads, f"{prefix}.w2", _wgrad(rl, dout))
    _acc(grads, f"{prefix}.b2", _sumto(dout, dout.shape[-1]))
    drl = np.matmul(dout, P[f"{prefix}.w2"].T) * (rl > 0)
    _acc(grads, f"{prefix}.w1", _wgrad(h, drl))
    _acc(grads, f"{prefix}.b1", _sumto(drl, drl.shape[-1]))
    dh = np.matmul(drl, P[f"{prefix}.w1"].T)
    dx, dg, db = ln_bwd(dh.astype(F32), ln_c)
    _acc(grads, f"{prefix}.ln_g", dg)
    _acc(grads, f"{prefix}.ln_b", db)
    return dout + dx


def opm_fwd(msa_in, msa_mask, P, prefix, k):
    """``outer_product_mean``, src/model.py:351-378 (serial: reduce-scatter = id)."""
    b, s, r, _ = msa_in.shape
    x, ln_c = ln_fwd(msa_in, P[f"{prefix}.ln_g"], P[f"{prefix}.ln_b"])
    mask4 = msa_mask.reshape(b, s, r, 1)
    a = (np.matmul(x, P[f"{prefix}.w_left"]) + P[f"{prefix}.b_left"]) * mask4
    c = (np.matmul(x, P[f"{prefix}.w_right"]) + P[f"{prefix}.b_right"]) * mask4
    af = np.ascontiguousarray(a.reshape(b, s, r * k).transpose(0, 2, 1))   # [1, rk, S]
    cf = c.reshape(b, s, r * k)
    num = np.matmul(af, cf)
    num = num.reshape(b, r, k, r, k).transpose(0, 1, 3, 2, 4).reshape(b, r, r, k * k)
    mt = np.ascontiguousarray(msa_mask.transpose(0, 2, 1))
    norm = np.matmul(mt, msa_mask).reshape(b, r, r, 1)
    rec = F32(1.0) / (norm + F32(1e-3))                               # recip (:375-376)
    outn = num * rec
    out = np.matmul(outn, P[f"{prefix}.w_out"]) + P[f"{prefix}.b_out"]
    return out.astype(F32), (ln_c, x, mask4, af, cf, rec, outn, (b, s, r, k))


def opm_bwd(dout, cache, P, prefix, grads):
    ln_c, x, mask4, af, cf, rec, outn, (b, s, r, k) = cache
    _acc(grads, f"{prefix}.w_out", _wgrad(outn, dout))
    _acc(grads, f"{prefix}.b_out", _sumto(dout, dout.shape[-1]))
    dnum = np.matmul(dout, P[f"{prefix}.w_out"].T) * rec
    dnum = dnum.reshape(b, r, r, k, k).transpose(0, 1, 3, 2, 4).reshape(b, r * k, r * k)
    daf = np.matmul(dnum, cf.swapaxes(-1, -2))                         # [1, rk, S]
    dcf = np.matmul(af.swapaxes(-1, -2), dnum)                         # [1, S, rk]
    da = daf.transpose(0, 2, 1).reshape(b, s, r, k) * mask4
    dc = dcf.reshape(b, s, r, k) * mask4
    _acc(grads, f"{prefix}.w_left", _wgrad(x, da))
    _acc(grads, f"{prefix}.b_left", _sumto(da, k))
    _acc(grads, f"{prefix}.w_right", _wgrad(x, dc))
    _acc(grads, f"{prefix}.b_right", _sumto(dc, k))
    dx = np.matmul(da, P[f"{prefix}.w_left"].T) + np.matmul(dc, P[f"{prefix}.w_right"].T)
    dmsa, dg, db = ln_bwd(dx.astype(F32), ln_c)
    _acc(grads, f"{prefix}.ln_g", dg)
    _acc(grads, f"{prefix}.ln_b", db)
    return dmsa


def tri_attn_fwd(pair, mask, P, prefix, ending):
    """``triangle_attention``, src/model.py:381-398 (serial).  ``mask`` is
    pair_mask for the starting node, pair_mask_t for the ending node."""
    z = np.ascontiguousarray(pair.transpose(0, 2, 1, 3)) if ending else pair
    x, ln_c = ln_fwd(z, P[f"{prefix}.ln_g"], P[f"{prefix}.ln_b"])
    nb, nb_c = pair_bias_fwd(z, P, prefix)
    y, a_c = attention_fwd(x, mask, nb, _attn_p(P, prefix))
    if ending:
        y = np.ascontiguousarray(y.transpose(0, 2, 1, 3))
    return pair + y, (ln_c, nb_c, a_c, ending)


def tri_attn_bwd(dout, cache, P, prefix, grads):
    ln_c, nb_c, a_c, ending = cache
    dy = np.ascontiguousarray(dout.transpose(0, 2, 1, 3)) if ending else dout
    dx, dp, dnb = attention_bwd(dy, a_c)
    _acc_attn(grads, prefix, dp)
    dz, dg, db = ln_bwd(dx, ln_c)
    _acc(grads, f"{prefix}.ln_g", dg)
    _acc(grads, f"{prefix}.ln_b", db)
    dz = dz + pair_bias_bwd(dnb, nb_c, P, prefix, grads)
    if ending:
        dz = np.ascontiguousarray(dz.transpose(0, 2, 1, 3))
    return dout + dz


# ---------------------------------------------------------------------------
# TriangleMultiplication -- EXTENSION, parity UNPINNED (no reference code).
# AF2 Supplementary Alg. 11 (outgoing) / Alg. 12 (incoming):
#   zl = LN(z); a = sigmoid(zl Wag + bag) * (zl Wap + bap) * mask
#   b likewise; outgoing o_ij = sum_k a_ik * b_jk; incoming o_ij = sum_k a_ki * b_kj
#   g = sigmoid(zl Wg + bg); z += g * (LN(o) Wo + bo)


def trimul_fwd(pair, pair_mask, P, prefix, outgoing):
    zl, ln_c = ln_fwd(pair, P[f"{prefix}.ln_in_g"], P[f"{prefix}.ln_in_b"])
    m = pair_mask[..., None]                                            # [1,R,R,1]
    ap = np.matmul(zl, P[f"{prefix}.w_ap"]) + P[f"{prefix}.b_ap"]
    ag = sigmoid(np.matmul(zl, P[f"{prefix}.w_ag"]) + P[f"{prefix}.b_ag"])
    bp = np.matmul(zl, P[f"{prefix}.w_bp"]) + P[f"{prefix}.b_bp"]
    bg = sigmoid(np.matmul(zl, P[f"{prefix}.w_bg"]) + P[f"{prefix}.b_bg"])
    a = (ag * ap * m).astype(F32)[0]                                    # [R,R,ch]
    bb = (bg * bp * m).astype(F32)[0]
    ac = np.ascontiguousarray(a.transpose(2, 0, 1))                     # [ch, R, R]
    bc = np.ascontiguousarray(bb.transpose(2, 0, 1))
    if outgoing:
        oc = np.matmul(ac, bc.swapaxes(-1, -2))                         # o_ij = a_ik b_jk
    else:
        oc = np.matmul(ac.swapaxes(-1, -2), bc)                         # o_ij = a_ki b_kj
    o = np.ascontiguousarray(oc.transpose(1, 2, 0))[None]               # [1,R,R,ch]
    ol, lno_c = ln_fwd(o, P[f"{prefix}.ln_out_g"], P[f"{prefix}.ln_out_b"])
    y = np.matmul(ol, P[f"{prefix}.w_o"]) + P[f"{prefix}.b_o"]
    g = sigmoid(np.matmul(zl, P[f"{prefix}.w_g"]) + P[f"{prefix}.b_g"])
    out = (pair + g * y).astype(F32)
    cache = (ln_c, zl, m, ap, ag, bp, bg, ac, bc, lno_c, ol, y, g, outgoing)
    return out, cache


def trimul_bwd(dout, cache, P, prefix, grads):
    ln_c, zl, m, ap, ag, bp, bg, ac, bc, lno_c, ol, y, g, outgoing = cache
    dy = dout * g
    dgl = dout * y * g * (F32(1.0) - g)
    _acc(grads, f"{prefix}.w_g", _wgrad(zl, dgl))
    _acc(grads, f"{prefix}.b_g", _sumto(dgl, dgl.shape[-1]))
    dzl = np.matmul(dgl, P[f"{prefix}.w_g"].T)
    _acc(grads, f"{prefix}.w_o", _wgrad(ol, dy))
    _acc(grads, f"{prefix}.b_o", _sumto(dy, dy.shape[-1]))
    dol = np.matmul(dy, P[f"{prefix}.w_o"].T)
    do, dg_, db_ = ln_bwd(dol.astype(F32), lno_c)
    _acc(grads, f"{prefix}.ln_out_g", dg_)
    _acc(grads, f"{prefix}.ln_out_b", db_)
    doc = np.ascontiguousarray(do[0].transpose(2, 0, 1))                # [ch, i, j]
    if outgoing:
        dac = np.matmul(doc, bc)                                        # da_ik = do_ij b_jk
        dbc = np.matmul(doc.swapaxes(-1, -2), ac)                       # db_jk = do_ij a_ik
    else:
        dac = np.matmul(bc, doc.swapaxes(-1, -2))                       # da_ki = b_kj do_ij
        dbc = np.matmul(ac, doc)                                        # db_kj = a_ki do_ij
    da = np.ascontiguousarray(dac.transpose(1, 2, 0))[None] * m
    db = np.ascontiguousarray(dbc.transpose(1, 2, 0))[None] * m
    dap, dagl = da * ag, da * ap * ag * (F32(1.0) - ag)
    dbp, dbgl = db * bg, db * bp * bg * (F32(1.0) - bg)
    for nm, d in (("ap", dap), ("ag", dagl), ("bp", dbp), ("bg", dbgl)):
        _acc(grads, f"{prefix}.w_{nm}", _wgrad(zl, d))
        _acc(grads, f"{prefix}.b_{nm}", _sumto(d, d.shape[-1]))
        dzl = dzl + np.matmul(d, P[f"{prefix}.w_{nm}"].T)
    dz, dg2, db2 = ln_bwd(dzl.astype(F32), ln_c)
    _acc(grads, f"{prefix}.ln_in_g", dg2)
    _acc(grads, f"{prefix}.ln_in_b", db2)
    return dout + dz


# ---------------------------------------------------------------------------
# block = two branches (src/model.py:431-445).  The split is the one branch
# parallelism uses (src/harness.py:447-486): the MSA branch reads
# (msa_in, pair_in); OPM reads msa_in; the pair branch reads pair_in + opm.


@dataclass
class Masks:
    msa: np.ndarray
    msa_t: np.ndarray
    pair: np.ndarray
    pair_t: np.ndarray


def make_masks(feats: Features) -> Masks:
    """src/model.py:421-428 (serial)."""
    mm, pm = feats.msa_mask, feats.pair_mask
    return Masks(mm, np.ascontiguousarray(mm.transpose(0, 2, 1)),
                 pm, np.ascontiguousarray(pm.transpose(0, 2, 1)))


def msa_branch_fwd(msa_in, pair_in, masks, P, i):
    p = f"block{i}"
    msa, c1 = row_attn_fwd(msa_in, pair_in, masks.msa, P, f"{p}.row_attn")
    msa, c2 = col_attn_fwd(msa, masks.msa_t, P, f"{p}.col_attn")
    msa, c3 = transition_fwd(msa, P, f"{p}.msa_trans")
    return msa, (c1, c2, c3)


def msa_branch_bwd(dmsa, cache, P, i, grads):
    """Returns (d msa_in, d pair_in) from the MSA branch."""
    p = f"block{i}"
    c1, c2, c3 = cache
    d = transition_bwd(dmsa, c3, P, f"{p}.msa_trans", grads)
    d = col_attn_bwd(d, c2, P, f"{p}.col_attn", grads)
    return row_attn_bwd(d, c1, P, f"{p}.row_attn", grads)


def pair_branch_fwd(pair_in, opm, masks, P, i, cfg=None):
    p = f"block{i}"
    pair = pair_in + opm
    caches = []
    if cfg is not None and cfg.trimul:
        pair, c = trimul_fwd(pair, masks.pair, P, f"{p}.tri_mul_out", True)
        caches.append(c)
        pair, c = trimul_fwd(pair, masks.pair, P, f"{p}.tri_mul_in", False)
        caches.append(c)
    pair, c1 = tri_attn_fwd(pair, masks.pair, P, f"{p}.tri_start", False)
    pair, c2 = tri_attn_fwd(pair, masks.pair_t, P, f"{p}.tri_end", True)
    pair, c3 = transition_fwd(pair, P, f"{p}.pair_trans")
    return pair, (caches, c1, c2, c3)


def pair_branch_bwd(dpair, cache, P, i, grads):
    """Returns d(pair_in + opm) (the same gradient flows to both)."""
    p = f"block{i}"
    tm, c1, c2, c3 = cache
    d = transition_bwd(dpair, c3, P, f"{p}.pair_trans", grads)
    d = tri_attn_bwd(d, c2, P, f"{p}.tri_end", grads)
    d = tri_attn_bwd(d, c1, P, f"{p}.tri_start", grads)
    if tm:
        d = trimul_bwd(d, tm[1], P, f"{p}.tri_mul_in", grads)
        d = trimul_bwd(d, tm[0], P, f"{p}.tri_mul_out", grads)
    return d


def block_fwd(msa_in, pair_in, masks, P, i, cfg):
    """``evoformer_block``, src/model.py:431-445."""
    msa, cm = msa_branch_fwd(msa_in, pair_in, masks, P, i)
    opm, co = opm_fwd(msa_in, masks.msa, P, f"block{i}.opm", cfg.opm_dim)
    pair, cp = pair_branch_fwd(pair_in, opm, masks, P, i, cfg)
    return msa, pair, (cm, co, cp)


def block_bwd(dmsa, dpair, cache, P, i, grads):
    cm, co, cp = cache
    dpm = pair_branch_bwd(dpair, cp, P, i, grads)
    dmsa_in2 = opm_bwd(dpm, co, P, f"block{i}.opm", grads)
    dmsa_in, dpair_in = msa_branch_bwd(dmsa, cm, P, i, grads)
    return dmsa_in + dmsa_in2, dpair_in + dpm


# ---------------------------------------------------------------------------
# trunk, loss and serial gradients (src/model.py:448-478, src/harness.py:313-357)


def embed_fwd(feats, P, prev=None):
    """``embed``, src/model.py:448-464."""
    msa = np.matmul(feats.msa_feat, P["msa_embed.w"]) + P["msa_embed.b"]
    pair = np.matmul(feats.pair_feat, P["pair_embed.w"]) + P["pair_embed.b"]
    rc = None
    if prev is not None:
        fb, cm = ln_fwd(prev[0][:, :1].copy(), P["recycle_m.g"], P["recycle_m.b"])
        msa = msa.copy()
        msa[:, :1] = msa[:, :1] + fb
        fz, cz = ln_fwd(prev[1].copy(), P["recycle_z.g"], P["recycle_z.b"])
        pair = pair + fz
        rc = (cm, cz)
    return msa.astype(F32), pair.astype(F32), rc


def embed_bwd(dmsa, dpair, feats, rc, grads):
    _acc(grads, "msa_embed.w", _wgrad(feats.msa_feat, dmsa))
    _acc(grads, "msa_embed.b", _sumto(dmsa, dmsa.shape[-1]))
    _acc(grads, "pair_embed.w", _wgrad(feats.pair_feat, dpair))
    _acc(grads, "pair_embed.b", _sumto(dpair, dpair.shape[-1]))
    if rc is not None:
        _, dg, db = ln_bwd(dmsa[:, :1], rc[0])
        _acc(grads, "recycle_m.g", dg)
        _acc(grads, "recycle_m.b", db)
        _, dg, db = ln_bwd(dpair, rc[1])
        _acc(grads, "recycle_z.g", dg)
        _acc(grads, "recycle_z.b", db)


def local_loss(cfg, msa, pair):
    """``_local_loss``, src/harness.py:313-320; returns (loss, dmsa, dpair)."""
    km = F32(1.0 / (cfg.n_seq * cfg.n_res * cfg.c_m))
    kz = F32(1.0 / (cfg.n_res * cfg.n_res * cfg.c_z))
    lm = F32(np.sum(msa * msa, dtype=F32)) * km
    lz = F32(np.sum(pair * pair, dtype=F32)) * kz
    return float(F32(lm + lz)), (km * msa) + (km * msa), (kz * pair) + (kz * pair)


def model_forward(cfg, P, feats, prev=None):
    """``model_forward``, src/model.py:467-472, untaped."""
    masks = make_masks(feats)
    msa, pair, _ = embed_fwd(feats, P, prev)
    for i in range(cfg.n_blocks):
        msa, pair, _ = block_fwd(msa, pair, masks, P, i, cfg)
    return msa, pair


def serial_grads(cfg, P, feats, n_cycles=1):
    """``_serial_grads``, src/harness.py:327-352: n-1 untaped recycles, then
    one differentiated pass.  Returns (loss, grads by name, (msa, pair))."""
    prev = None
    for _ in range(max(0, n_cycles - 1)):
        prev = model_forward(cfg, P, feats, prev)
    masks = make_masks(feats)
    msa, pair, rc = embed_fwd(feats, P, prev)
    caches = []
    for i in range(cfg.n_blocks):
        msa, pair, c = block_fwd(msa, pair, masks, P, i, cfg)
        caches.append(c)
    loss, dmsa, dpair = local_loss(cfg, msa, pair)
    grads = {}
    for i in reversed(range(cfg.n_blocks)):
        dmsa, dpair = block_bwd(dmsa, dpair, caches[i], P, i, grads)
    embed_bwd(dmsa, dpair, feats, rc, grads)
    out = {name: grads.get(name, np.zeros(shape, F32)).astype(F32)
           for name, shape, _ in param_specs(cfg)}
    return loss, out, (msa, pair)


def serial_grads_f64(cfg, P, feats, n_cycles=1):
    """``serial_grads`` evaluated in float64 (inputs and parameters are the
    fp32 ones, promoted; the fp32 rounding of the masked logits is kept).  The
    fp32 restatement's own deviation from this bounds what any fp32
    implementation can be expected to match it to: long reductions at the
    initial-training shape (65,536-term weight gradients, 128-sequence bias
    gradients) leave ~1e-4 relative rounding in a few small gradients."""
    global F32
    saved = F32
    F32 = np.float64
    try:
        P64 = {k: np.asarray(v, np.float64) for k, v in P.items()}
        f64 = Features(**{k: np.asarray(getattr(feats, k), np.float64)
                          for k in ("msa_feat", "pair_feat", "msa_mask", "pair_mask")})
        return serial_grads(cfg, P64, f64, n_cycles)
    finally:
        F32 = saved


# ---------------------------------------------------------------------------
# tensor fusion + optimizer tail (src/fusion.py:27-237)

ALIGN = 256


@dataclass
class OptimConfig:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    clip_norm: float = 0.1
    ema_decay: float = 0.999


def build_layout(named_shapes, align=ALIGN):
    """src/fusion.py:50-58: [(name, shape, byte offset, nbytes, padded)]."""
    out, off = [], 0
    for name, shape in named_shapes:
        nbytes = int(np.prod(shape, dtype=np.int64)) * 4 if shape else 4
        padded = -(-nbytes // align) * align
        out.append((name, tuple(shape), off, nbytes, padded))
        off += padded
    return out


@dataclass
class FusedOptimizer:
    """Fused-mode ``FusionEngine`` numerics, src/fusion.py:142-233."""

    params: dict
    optim: OptimConfig = field(default_factory=OptimConfig)
    step_count: int = 0

    def __post_init__(self):
        self.m = {n: np.zeros_like(v) for n, v in self.params.items()}
        self.v = {n: np.zeros_like(v) for n, v in self.params.items()}
        self.ema = {n: v.copy() for n, v in self.params.items()}

    def apply(self, grads: dict) -> float:
        o = self.optim
        names = list(self.params)
        acc = np.float64(0.0)                                           # :164-171
        for n in names:
            g = np.asarray(grads[n], np.float64).ravel()
            acc += np.dot(g, g)
        norm = float(np.sqrt(acc))
        scale = F32(1.0)
        if norm > o.clip_norm:                                          # :173-187
            scale = F32(o.clip_norm / norm)
        self.step_count += 1                                            # :189-211
        t = self.step_count
        bc1 = F32(1.0 - o.beta1 ** t)
        bc2 = F32(1.0 - o.beta2 ** t)
        d = F32(o.ema_decay)
        for n in names:
            g = np.asarray(grads[n], F32).reshape(self.params[n].shape)
            if scale != 1.0:
                g = g * scale
            m, v, p = self.m[n], self.v[n], self.params[n]
            m[...] = F32(o.beta1) * m + F32(1 - o.beta1) * g
            v[...] = F32(o.beta2) * v + F32(1 - o.beta2) * (g * g)
            p -= F32(o.lr) * (m / bc1) / (np.sqrt(v / bc2) + F32(o.eps))
            self.ema[n][...] = d * self.ema[n] + (F32(1.0) - d) * p     # :213-224
        return norm
