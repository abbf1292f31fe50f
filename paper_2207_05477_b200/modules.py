"""The reference block-module API (src/model.py:140-478) on torch CUDA tensors.

Same names, parameter dataclasses and argument meaning as ``evotrain.model``:

  ``init_params`` / ``flatten_params`` / ``branch_param_names``  (src/model.py:172-236)
  ``SerialPar``                                                  (src/model.py:243-259)
  ``_run_attention`` (+ ``subbatch_apply`` for ``row_chunk``)     (src/model.py:300-309)
  ``_pair_bias``                                                 (src/model.py:312-317)
  ``msa_row_attention`` / ``msa_col_attention``                  (src/model.py:320-341)
  ``transition`` / ``outer_product_mean``                        (src/model.py:344-378)
  ``triangle_attention`` (starting / ending)                     (src/model.py:381-398)
  ``TrackState`` / ``Masks`` / ``make_masks``                    (src/model.py:404-428)
  ``evoformer_block`` / ``embed`` / ``model_forward`` / ``model_loss`` (src/model.py:431-478)

Activations are torch tensors in the reference's shapes (msa ``[1, S, R, c_m]``,
pair ``[1, R, R, c_z]``, masks ``[1, S, R]`` / ``[1, R, S]`` / ``[1, R, R]``);
parameters are fp32 leaf tensors (``requires_grad`` as the caller likes) in
the reference's shapes.  Every function is a ``torch.autograd.Function``
that is a thin call into the block engine's kernels (``engine.BlockEngine``:
the same code paths the trainer and the bench run), so torch autograd is
only the shell: forward and backward arithmetic is the library's.

Activation dtype.  The reference rounds op outputs to bf16 when its runtime
context says so (src/tensor.py:102-108, ``Context.act_dtype``).  Here the
module functions compute in the dtype of their activation inputs (fp32 or
bf16 storage, fp32 math); ``embed`` -- the one module whose inputs are
host features -- takes it from ``act_dtype()`` (a thread-local mirror of the
reference's context, set with ``set_act_dtype`` or the ``activation_dtype``
context manager).

Sharding.  Only the serial adapter is supported at this level (``par.size``
must be 1); the sharded paths are ``parallel.bp_step`` / ``dap.DapEngine``.
"""

from __future__ import annotations

import contextlib
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .attention import (AttentionInput, AttentionParams, gated_attention_fused,
                        gated_attention_reference, subbatch_apply)
from .engine import BlockEngine, Variant, variants
from .errors import ContractError, DimensionError
from .model import (MSA_BRANCH_MODULES, PAIR_BRANCH_MODULES, TRIMUL_MODULES, ExecPolicy, Features,
                    ModelConfig, draw_num_recycles, make_features)
from .model import init_params as _init_flat
from .model import param_specs

F32 = torch.float32
BF16 = torch.bfloat16

__all__ = [
    "AttnModuleParams", "TransitionParams", "OpmParams", "TriMulParams", "BlockParams", "ModelParams",
    "TrackState", "Masks", "SerialPar", "ExecPolicy", "ModelConfig", "Features", "AttentionInput",
    "AttentionParams", "init_params", "flatten_params", "branch_param_names", "make_features",
    "make_masks", "draw_num_recycles", "_run_attention", "_pair_bias", "msa_row_attention",
    "msa_col_attention", "transition", "outer_product_mean", "triangle_attention",
    "triangle_multiplication", "evoformer_block", "embed", "model_forward", "model_loss",
    "act_dtype", "set_act_dtype", "activation_dtype", "subbatch_apply",
]


# --------------------------------------------------------------------------
# activation-dtype context (mirror of src/runtime.py Context.act_dtype)

_ctx = threading.local()


def act_dtype() -> torch.dtype:
    return getattr(_ctx, "dtype", F32)


def set_act_dtype(dtype) -> None:
    if dtype is None:
        dtype = F32
    if dtype not in (F32, BF16):
        raise ContractError(f"activation dtype must be float32 or bfloat16, got {dtype}")
    _ctx.dtype = dtype


@contextlib.contextmanager
def activation_dtype(dtype):
    prev = act_dtype()
    set_act_dtype(dtype)
    try:
        yield
    finally:
        set_act_dtype(prev)


# --------------------------------------------------------------------------
# parameter dataclasses (src/model.py:76-130)


@dataclass
class AttnModuleParams:
    ln_g: torch.Tensor
    ln_b: torch.Tensor
    attn: AttentionParams
    bias_ln_g: torch.Tensor = None  # present when a pair-derived bias is used
    bias_ln_b: torch.Tensor = None
    w_bias: torch.Tensor = None  # [C_z, H]


@dataclass
class TransitionParams:
    ln_g: torch.Tensor
    ln_b: torch.Tensor
    w1: torch.Tensor
    b1: torch.Tensor
    w2: torch.Tensor
    b2: torch.Tensor


@dataclass
class OpmParams:
    ln_g: torch.Tensor
    ln_b: torch.Tensor
    w_left: torch.Tensor  # [C_m, k]
    b_left: torch.Tensor
    w_right: torch.Tensor
    b_right: torch.Tensor
    w_out: torch.Tensor  # [k*k, C_z]
    b_out: torch.Tensor


@dataclass
class TriMulParams:
    """TriangleMultiplication (extension, AF2 Alg 11/12; not in the reference)."""

    ln_in_g: torch.Tensor
    ln_in_b: torch.Tensor
    w_ap: torch.Tensor
    b_ap: torch.Tensor
    w_ag: torch.Tensor
    b_ag: torch.Tensor
    w_bp: torch.Tensor
    b_bp: torch.Tensor
    w_bg: torch.Tensor
    b_bg: torch.Tensor
    ln_out_g: torch.Tensor
    ln_out_b: torch.Tensor
    w_o: torch.Tensor
    b_o: torch.Tensor
    w_g: torch.Tensor
    b_g: torch.Tensor


@dataclass
class BlockParams:
    row_attn: AttnModuleParams
    col_attn: AttnModuleParams
    msa_trans: TransitionParams
    opm: OpmParams
    tri_start: AttnModuleParams
    tri_end: AttnModuleParams
    pair_trans: TransitionParams
    tri_mul_out: TriMulParams = None
    tri_mul_in: TriMulParams = None


@dataclass
class ModelParams:
    msa_embed_w: torch.Tensor
    msa_embed_b: torch.Tensor
    pair_embed_w: torch.Tensor
    pair_embed_b: torch.Tensor
    recycle_m_g: torch.Tensor
    recycle_m_b: torch.Tensor
    recycle_z_g: torch.Tensor
    recycle_z_b: torch.Tensor
    blocks: list = field(default_factory=list)


_EMBED = (("msa_embed.w", "msa_embed_w"), ("msa_embed.b", "msa_embed_b"),
          ("pair_embed.w", "pair_embed_w"), ("pair_embed.b", "pair_embed_b"),
          ("recycle_m.g", "recycle_m_g"), ("recycle_m.b", "recycle_m_b"),
          ("recycle_z.g", "recycle_z_g"), ("recycle_z.b", "recycle_z_b"))
_ATTN = ("wq", "wk", "wv", "wg", "bg", "wo", "bo")


def _module_named(sub, prefix: str) -> list:
    """[(flatten name, tensor)] of one module dataclass in the reference's
    field order (src/model.py:207-219); absent optional fields are skipped."""
    out = []
    for fname in sub.__dataclass_fields__:
        t = getattr(sub, fname)
        if t is None:
            continue
        if isinstance(t, AttentionParams):
            out += [(f"{prefix}.attn.{a}", getattr(t, a)) for a in _ATTN]
        else:
            out.append((f"{prefix}.{fname}", t))
    return out


def _from_flat(cfg: ModelConfig, flat: dict) -> ModelParams:
    def attn_mod(p, bias):
        ap = AttentionParams(*[flat[f"{p}.attn.{a}"] for a in _ATTN])
        m = AttnModuleParams(flat[f"{p}.ln_g"], flat[f"{p}.ln_b"], ap)
        if bias:
            m.bias_ln_g, m.bias_ln_b, m.w_bias = (flat[f"{p}.bias_ln_g"], flat[f"{p}.bias_ln_b"],
                                                  flat[f"{p}.w_bias"])
        return m

    def trans(p):
        return TransitionParams(*[flat[f"{p}.{f}"] for f in ("ln_g", "ln_b", "w1", "b1", "w2", "b2")])

    mp = ModelParams(*[flat[n] for n, _ in _EMBED])
    for i in range(cfg.n_blocks):
        p = f"block{i}"
        blk = BlockParams(
            row_attn=attn_mod(f"{p}.row_attn", True), col_attn=attn_mod(f"{p}.col_attn", False),
            msa_trans=trans(f"{p}.msa_trans"),
            opm=OpmParams(*[flat[f"{p}.opm.{f}"] for f in OpmParams.__dataclass_fields__]),
            tri_start=attn_mod(f"{p}.tri_start", True), tri_end=attn_mod(f"{p}.tri_end", True),
            pair_trans=trans(f"{p}.pair_trans"))
        if cfg.trimul:
            for m in TRIMUL_MODULES:
                setattr(blk, m, TriMulParams(*[flat[f"{p}.{m}.{f}"] for f in TriMulParams.__dataclass_fields__]))
        mp.blocks.append(blk)
    return mp


def init_params(cfg: ModelConfig, seed: int, device="cuda", requires_grad: bool = True) -> ModelParams:
    """src/model.py:172-200: the reference's splitmix64 draws (bit-identical
    to ``model.init_params``) as fp32 leaf tensors on ``device``."""
    flat = {n: torch.from_numpy(np.ascontiguousarray(v)).to(device).requires_grad_(requires_grad)
            for n, v in _init_flat(cfg, seed).items()}
    return _from_flat(cfg, flat)


def flatten_params(mp: ModelParams) -> list:
    """src/model.py:203-220: deterministic (name, tensor) order (the fusion
    engine's slot order)."""
    out = [(n, getattr(mp, a)) for n, a in _EMBED]
    for i, blk in enumerate(mp.blocks):
        for mod in MSA_BRANCH_MODULES + PAIR_BRANCH_MODULES + TRIMUL_MODULES:
            sub = getattr(blk, mod)
            if sub is not None:
                out += _module_named(sub, f"block{i}.{mod}")
    return out


def branch_param_names(mp: ModelParams, branch: str) -> set:
    """src/model.py:223-236 (TriMul, when present, is pair-branch)."""
    embeds = {"msa": ("msa_embed.", "recycle_m."), "pair": ("pair_embed.", "recycle_z.")}[branch]
    mods = MSA_BRANCH_MODULES if branch == "msa" else PAIR_BRANCH_MODULES + TRIMUL_MODULES
    return {n for n, _ in flatten_params(mp)
            if n.startswith(embeds) or (n.startswith("block") and n.split(".")[1] in mods)}


class SerialPar:
    """src/model.py:243-259: identity adapter, every collective a no-op."""

    size = 1
    index = 0

    def slice_np(self, arr, axis: int):
        return arr

    def allgather(self, x, axis: int, module: str):
        return x

    def reducescatter_sum(self, x, axis: int, module: str):
        return x

    def alltoall(self, x, split_axis: int, concat_axis: int, module: str):
        return x


def _serial(par):
    if par is not None and getattr(par, "size", 1) != 1:
        raise ContractError("the module API runs the serial adapter only; sharded runs go through "
                            "parallel.bp_step / dap.DapEngine")


# --------------------------------------------------------------------------
# engine adapter: a FusionEngine-shaped view over one module's tensors


class _ModuleStore:
    """What ``BlockEngine`` reads from its parameter store (``param`` fp32,
    ``weight`` = the projection operand in the activation dtype, ``grad``
    fp32 written by the kernels), over the caller's tensors: fp32
    contiguous params are used in place (no copy)."""

    def __init__(self, named, dt):
        named = list(named)
        self.device = named[0][1].device
        self.p, self.g, self.w = {}, {}, {}
        for n, t in named:
            p = t.detach()
            if p.dtype != F32:
                raise TypeError(f"parameter {n} must be float32, got {p.dtype}")
            p = p.contiguous()
            self.p[n] = p
            self.g[n] = torch.zeros_like(p)
            if dt == F32:
                self.w[n] = p
            else:
                w = torch.empty(p.shape, dtype=dt, device=p.device)
                self.w[n] = ops.cast(p, w)

    def param(self, n):
        return self.p[n]

    def grad(self, n):
        return self.g[n]

    def weight(self, n):
        return self.w[n]

    def zero_grads(self):
        for g in self.g.values():
            g.zero_()


class _Feats:
    """DeviceFeatures-shaped holder of fp32 flat masks (and features)."""

    def __init__(self, msa_mask=None, pair_mask=None, msa_feat=None, pair_feat=None):
        self.msa_mask, self.pair_mask = msa_mask, pair_mask
        self.msa_feat, self.pair_feat = msa_feat, pair_feat


def _flat_mask(m, n, dev):
    m = torch.as_tensor(np.asarray(m, np.float32)) if not isinstance(m, torch.Tensor) else m
    if m.numel() != n:
        raise DimensionError(f"mask has {m.numel()} elements, want {n}")
    m = m.detach().to(dev).reshape(n)
    if m.dtype != F32:
        m = ops.cast(m.contiguous(), torch.empty(n, dtype=F32, device=dev))
    return m.contiguous()


def _engine(cfg0: ModelConfig, store: _ModuleStore, dt, arena_mb: int = 0, streams: bool = False):
    eng = BlockEngine(cfg0, store, dt, arena_mb=arena_mb)
    eng.branch_streams = streams and eng.branch_streams
    return eng


def _pack(eng, store, prefix, names, C, N, dt):
    """Merged projection operand [C, len(names)*N] (the engine's wcat)."""
    buf = torch.empty((C, len(names) * N), dtype=dt, device=store.device)
    plan = ops.PackPlan([store.weight(n) for n in names], [buf], [C], [N], False,
                        ops.dcode(store.weight(names[0])), ops.dcode(buf), ns=len(names))
    plan.run()
    eng.wcat[prefix] = buf


def _act(x, what):
    if not isinstance(x, torch.Tensor) or x.dtype not in (F32, BF16):
        raise TypeError(f"{what} must be a float32 or bfloat16 torch tensor")
    if x.dim() != 4 or x.shape[0] != 1:
        raise DimensionError(f"{what} shape {tuple(x.shape)}, want [1, *, *, C]")
    return x


def _f32_copy(t, shape):
    out = torch.empty(shape, dtype=F32, device=t.device)
    return ops.cast(t.detach().contiguous().reshape(shape), out)


def _to_dtype(t, dt):
    if t.dtype == dt:
        return t
    return ops.cast(t, torch.empty(t.shape, dtype=dt, device=t.device))


class _EngineOp(torch.autograd.Function):
    """Generic shell: ``job.fwd(*tensors)`` -> outputs, ``job.bwd(*gouts)`` ->
    one gradient (or None) per input tensor."""

    @staticmethod
    def forward(ctx, job, *ts):
        ctx.job = job
        out = job.fwd(*ts)
        if isinstance(out, tuple):
            ctx.mark_non_differentiable(*[o for o, d in zip(out, job.differentiable) if not d])
        return out

    @staticmethod
    def backward(ctx, *gouts):
        job, ctx.job = ctx.job, None
        return (None, *job.bwd(*gouts))


def _params_grads(store, named):
    return [store.g[n].view(t.shape) for n, t in named]


# --------------------------------------------------------------------------
# attention modules (src/model.py:300-328, 331-341, 381-398)


class _AttnJob:
    """LayerNorm -> [pair bias] -> fused gated attention -> residual, on one
    attention geometry (engine.Variant)."""

    def __init__(self, kind, mod: AttnModuleParams, has_pair: bool):
        self.kind, self.has_pair = kind, has_pair
        self.named = _module_named(mod, "m")

    def fwd(self, x4, pair4, mask, *params):
        x4 = x4.contiguous()
        pair4 = pair4.contiguous() if pair4 is not None else None
        _, A, Bn, C = x4.shape
        dt = x4.dtype
        H, D = params[2].shape[1], params[2].shape[2]
        if H * D != C:
            raise DimensionError(f"x channels {C} vs wq {tuple(params[2].shape)}")
        x2 = x4.reshape(A * Bn, C)
        self.store = st = _ModuleStore(self.named, dt)
        R = Bn if self.kind in ("row", "tri_start", "tri_end") else A
        S = A if self.kind == "row" else (Bn if self.kind == "col" else R)
        cz = pair4.shape[-1] if pair4 is not None else C
        self.cfg0 = ModelConfig(n_blocks=0, n_seq=S, n_res=R, c_m=C, c_z=cz, heads=H)
        self.eng = eng = _engine(self.cfg0, st, dt)
        _pack(eng, st, "m", [f"m.attn.{w}" for w in ("wq", "wk", "wv", "wg")], C, H * D, dt)
        n = A * Bn
        if self.kind == "row":      # batch s, keys r, mask msa[s, r]
            v = Variant("row_attn", A, Bn, Bn, 1, Bn, 1, "msa", True, False)
            self.feats = _Feats(msa_mask=_flat_mask(mask, n, x4.device))
        elif self.kind == "col":    # msa [1, S, R, C]; batch r, keys s, mask_t[r, s]
            v = Variant("col_attn", Bn, A, 1, Bn, A, 1, "msa", False, False)
            self.feats = _Feats(msa_mask=_flat_mask(mask, n, x4.device))
        elif self.kind == "tri_start":  # batch i, keys j, mask pair[i, j]
            v = Variant("tri_start", A, Bn, Bn, 1, Bn, 1, "pair", True, False)
            self.feats = _Feats(pair_mask=_flat_mask(mask, n, x4.device))
        else:                       # batch j of pair^T, keys i, mask pair_t[j, i]
            v = Variant("tri_end", A, Bn, 1, Bn, Bn, 1, "pair", True, True)
            self.feats = _Feats(pair_mask=_flat_mask(mask, n, x4.device))
        self.v = v
        pair2 = None
        if self.has_pair:
            if pair4.dtype != dt:
                raise TypeError("msa and pair must share the activation dtype")
            pair2 = pair4.reshape(-1, cz)
            self.pair_shape = pair4.shape
        out, self.saved = eng.attn_fwd(x2, "m", v, self.feats, pair=pair2)
        self.x_shape, self.dt = x4.shape, dt
        return out.view(x4.shape)

    @property
    def differentiable(self):
        return (True,)

    def bwd(self, gout):
        _, A, Bn, C = self.x_shape
        d = _f32_copy(gout, (A * Bn, C))
        dpair = None
        if self.has_pair:
            dpair = torch.zeros((self.pair_shape[1] * self.pair_shape[2], self.pair_shape[3]), dtype=F32,
                                device=d.device)
        self.eng.attn_bwd(d, self.saved, "m", self.v, self.feats, dpair=dpair)
        self.saved = None
        dx = _to_dtype(d, self.dt).view(self.x_shape)
        dp = _to_dtype(dpair, self.dt).view(self.pair_shape) if dpair is not None else None
        return (dx, dp, None, *_params_grads(self.store, self.named))


def _attn_module(kind, x, pair, mask, mod: AttnModuleParams):
    job = _AttnJob(kind, mod, pair is not None)
    params = [t for _, t in job.named]
    return _EngineOp.apply(job, _act(x, "x"), None if pair is None else _act(pair, "pair"), mask, *params)


def _run_attention(inp: AttentionInput, p: AttentionParams, policy: ExecPolicy, chunk: int = 0):
    """src/model.py:300-309: the fused operator, or with ``policy.fused``
    False the unfused fp32 baseline (materialised logits), chunked over dim 1
    with the mask as companion and the bias shared when ``chunk`` > 0."""
    dt = inp.x.dtype if inp.x.dtype in (F32, BF16) else F32
    if policy.fused:
        f = gated_attention_fused
    else:
        def f(i, pp, act_dtype=None):  # the baseline computes in fp32 (src/attention.py:78-115)
            return gated_attention_reference(i, pp)
    if chunk:
        nb = inp.nonbatched_bias
        return subbatch_apply(lambda xc, mc: f(AttentionInput(xc, mc, nb), p, act_dtype=dt),
                              inp.x, 1, chunk, companions=(inp.mask,))
    return f(inp, p, act_dtype=dt)


class _PairBiasJob:
    def __init__(self, mod: AttnModuleParams):
        self.named = [("m.bias_ln_g", mod.bias_ln_g), ("m.bias_ln_b", mod.bias_ln_b), ("m.w_bias", mod.w_bias)]

    differentiable = (True,)

    def fwd(self, z4, g, b, w):
        z4 = z4.contiguous()
        _, ni, nj, C = z4.shape
        H = w.shape[1]
        self.shape, self.dt, self.H = z4.shape, z4.dtype, H
        self.store = st = _ModuleStore(self.named, z4.dtype)
        self.z = z4.reshape(ni * nj, C)
        nb, self.mu, self.rs = ops.pair_bias_fwd(self.z, st.p["m.bias_ln_g"], st.p["m.bias_ln_b"],
                                                 st.p["m.w_bias"], ni, H, False, ni=ni, nj=nj)
        return nb

    def bwd(self, dnb):
        _, ni, nj, C = self.shape
        st = self.store
        dnb = _f32_copy(dnb, (self.H, ni, nj))
        dz = torch.zeros((ni * nj, C), dtype=F32, device=dnb.device)
        ops.pair_bias_bwd(self.z, self.mu, self.rs, st.p["m.bias_ln_g"], st.p["m.bias_ln_b"], st.p["m.w_bias"],
                          dnb, False, dz, st.g["m.bias_ln_g"], st.g["m.bias_ln_b"], st.g["m.w_bias"], ni,
                          self.H, ni=ni, nj=nj)
        return (_to_dtype(dz, self.dt).view(self.shape), *_params_grads(st, self.named))


def _pair_bias(pair, mod: AttnModuleParams, par=None, axis: int = 1, module: str = ""):
    """src/model.py:312-317: nb[h, i, j] = sum_c LN(z)[i, j, c] w_bias[c, h]
    as [H, r_local, R] (the LayerNorm is folded into the projection)."""
    _serial(par)
    job = _PairBiasJob(mod)
    return _EngineOp.apply(job, _act(pair, "pair"), *[t for _, t in job.named])


def msa_row_attention(msa, pair, msa_mask, blk: BlockParams, par=None, policy: ExecPolicy = None):
    """src/model.py:320-328: msa + Attn(LN(msa), msa_mask, nb=_pair_bias(pair));
    ``policy.row_chunk`` > 0 chunks the rows (the bias is recomputed per
    chunk; outputs equal the unchunked call)."""
    _serial(par)
    policy = policy or ExecPolicy()
    mod = blk.row_attn
    if policy.row_chunk and policy.row_chunk < msa.shape[1]:
        return subbatch_apply(lambda xc, mc: _attn_module("row", xc, pair, mc, mod), msa, 1, policy.row_chunk,
                              companions=(torch.as_tensor(msa_mask),))
    return _attn_module("row", msa, pair, msa_mask, mod)


def msa_col_attention(msa, msa_mask_t, blk: BlockParams, par=None, policy: ExecPolicy = None):
    """src/model.py:331-341: column attention over S with the transposed mask
    ``[1, R, S]``; read by stride, so no transposes run."""
    _serial(par)
    return _attn_module("col", msa, None, msa_mask_t, blk.col_attn)


def triangle_attention(pair, pair_mask, mod: AttnModuleParams, par=None, policy: ExecPolicy = None,
                       ending: bool = False):
    """src/model.py:381-398: ``pair_mask`` is the pair mask (starting) or its
    transpose (ending), as in the reference's ``Masks``."""
    _serial(par)
    return _attn_module("tri_end" if ending else "tri_start", pair, None, pair_mask, mod)


# --------------------------------------------------------------------------
# transition (src/model.py:344-348)


class _TransJob:
    differentiable = (True,)

    def __init__(self, tp: TransitionParams):
        self.named = _module_named(tp, "m")

    def fwd(self, x4, *params):
        x4 = x4.contiguous()
        _, A, Bn, C = x4.shape
        dt = x4.dtype
        self.store = st = _ModuleStore(self.named, dt)
        self.eng = _engine(ModelConfig(n_blocks=0, n_seq=A, n_res=Bn, c_m=C, c_z=C, heads=1), st, dt)
        out, self.saved = self.eng.trans_fwd(x4.reshape(A * Bn, C), "m")
        self.shape, self.dt = x4.shape, dt
        return out.view(x4.shape)

    def bwd(self, gout):
        _, A, Bn, C = self.shape
        d = _f32_copy(gout, (A * Bn, C))
        self.eng.trans_bwd(d, self.saved, "m")
        self.saved = None
        return (_to_dtype(d, self.dt).view(self.shape), *_params_grads(self.store, self.named))


def transition(x, tp: TransitionParams):
    """src/model.py:344-348: x + relu(LN(x) W1 + b1) W2 + b2."""
    job = _TransJob(tp)
    return _EngineOp.apply(job, _act(x, "x"), *[t for _, t in job.named])


# --------------------------------------------------------------------------
# outer product mean (src/model.py:351-378)


class _OpmJob:
    differentiable = (True,)

    def __init__(self, op: OpmParams):
        self.named = _module_named(op, "m")

    def fwd(self, msa4, mask, *params):
        msa4 = msa4.contiguous()
        _, S, R, Cm = msa4.shape
        dt = msa4.dtype
        k = params[2].shape[1]
        cz = params[6].shape[1]
        if params[6].shape[0] != k * k:
            raise DimensionError(f"w_out {tuple(params[6].shape)} vs opm_dim {k}")
        self.store = st = _ModuleStore(self.named, dt)
        cfg0 = ModelConfig(n_blocks=0, n_seq=S, n_res=R, c_m=Cm, c_z=cz, heads=1, opm_dim=k)
        self.eng = eng = _engine(cfg0, st, dt)
        _pack(eng, st, "m", ["m.w_left", "m.w_right"], Cm, k, dt)
        self.feats = _Feats(msa_mask=_flat_mask(mask, S * R, msa4.device))
        out, self.saved = eng.opm_fwd(msa4.reshape(S * R, Cm), "m", self.feats)
        self.shape, self.dt, self.oshape = msa4.shape, dt, (1, R, R, cz)
        return out.view(self.oshape)

    def bwd(self, gout):
        _, S, R, Cm = self.shape
        d = _f32_copy(gout, (R * R, self.oshape[3]))
        dxl = self.eng.opm_bwd_core(d, self.saved, "m", self.feats)
        d_msa = torch.zeros((S * R, Cm), dtype=F32, device=d.device)
        self.eng.opm_ln_bwd(dxl, self.saved, "m", d_msa)
        self.saved = None
        return (_to_dtype(d_msa, self.dt).view(self.shape), None, *_params_grads(self.store, self.named))


def outer_product_mean(msa_in, msa_mask, op: OpmParams, par=None, cfg: ModelConfig = None):
    """src/model.py:351-378: (a^T c over sequences, p-major flatten) /
    (mask^T mask + 1e-3) -> w_out; a = (LN(m) Wl + bl) * mask, c likewise."""
    _serial(par)
    job = _OpmJob(op)
    return _EngineOp.apply(job, _act(msa_in, "msa_in"), msa_mask, *[t for _, t in job.named])


# --------------------------------------------------------------------------
# TriangleMultiplication (extension: AF2 Alg 11/12, not in the reference)


class _TriMulJob:
    differentiable = (True,)

    def __init__(self, tp: TriMulParams, outgoing: bool):
        self.named = _module_named(tp, "m")
        self.outgoing = outgoing

    def fwd(self, z4, mask, *params):
        z4 = z4.contiguous()
        _, R, R2, Cz = z4.shape
        dt = z4.dtype
        ch = params[2].shape[1]
        self.store = st = _ModuleStore(self.named, dt)
        cfg0 = ModelConfig(n_blocks=0, n_seq=1, n_res=R, c_m=Cz, c_z=Cz, heads=1, trimul=True,
                           trimul_hidden=ch)
        self.eng = eng = _engine(cfg0, st, dt)
        _pack(eng, st, "m", [f"m.w_{n}" for n in ("ap", "ag", "bp", "bg")], Cz, ch, dt)
        self.feats = _Feats(pair_mask=_flat_mask(mask, R * R, z4.device))
        out, self.saved = eng.trimul_fwd(z4.reshape(R * R, Cz), "m", self.feats, self.outgoing)
        self.shape, self.dt = z4.shape, dt
        return out.view(z4.shape)

    def bwd(self, gout):
        _, R, _, Cz = self.shape
        d = _f32_copy(gout, (R * R, Cz))
        self.eng.trimul_bwd(d, self.saved, "m", self.feats)
        self.saved = None
        return (_to_dtype(d, self.dt).view(self.shape), None, *_params_grads(self.store, self.named))


def triangle_multiplication(pair, pair_mask, tp: TriMulParams, outgoing: bool = True):
    """pair + sigma(LN(z) Wg) * (LN(o) Wo + bo): o_ij = sum_k a_ik b_jk
    (outgoing) or sum_k a_ki b_kj (incoming) -- extension, parity unpinned."""
    job = _TriMulJob(tp, outgoing)
    return _EngineOp.apply(job, _act(pair, "pair"), pair_mask, *[t for _, t in job.named])


# --------------------------------------------------------------------------
# block / trunk (src/model.py:404-478)


@dataclass
class TrackState:
    msa: torch.Tensor  # [1, S, R, C_m]
    pair: torch.Tensor  # [1, R, R, C_z]


@dataclass
class Masks:
    """Mask tensors on the device (src/model.py:412-428)."""

    msa: torch.Tensor    # [1, S, R]
    msa_t: torch.Tensor  # [1, R, S]
    pair: torch.Tensor   # [1, R, R]
    pair_t: torch.Tensor


def make_masks(feats: Features, par=None, device="cuda") -> Masks:
    _serial(par)
    mm = np.asarray(feats.msa_mask, np.float32)
    pm = np.asarray(feats.pair_mask, np.float32)

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return Masks(up(mm), up(mm.transpose(0, 2, 1)), up(pm), up(pm.transpose(0, 2, 1)))


class _BlockJob:
    """One whole Evoformer block on the engine (``block_fwd`` / ``block_bwd``:
    the trainer's path, with the MSA branch on a second stream)."""

    def __init__(self, blk: BlockParams):
        self.named = []
        for mod in MSA_BRANCH_MODULES + PAIR_BRANCH_MODULES + TRIMUL_MODULES:
            sub = getattr(blk, mod)
            if sub is not None:
                self.named += _module_named(sub, f"block0.{mod}")
        self.trimul = blk.tri_mul_out is not None
        self.differentiable = (True, True)

    def fwd(self, msa4, pair4, msa_mask, pair_mask, *params):
        msa4, pair4 = msa4.contiguous(), pair4.contiguous()
        _, S, R, Cm = msa4.shape
        Cz = pair4.shape[3]
        dt = msa4.dtype
        if pair4.dtype != dt:
            raise TypeError("msa and pair must share the activation dtype")
        blk_named = dict(self.named)
        H = blk_named["block0.row_attn.attn.wq"].shape[1]
        k = blk_named["block0.opm.w_left"].shape[1]
        ch = blk_named["block0.tri_mul_out.w_ap"].shape[1] if self.trimul else 0
        cfg0 = ModelConfig(n_blocks=1, n_seq=S, n_res=R, c_m=Cm, c_z=Cz, heads=H, opm_dim=k,
                           trimul=self.trimul, trimul_hidden=ch)
        self.store = st = _ModuleStore(self.named, dt)
        self.eng = eng = _engine(cfg0, st, dt)
        self.feats = _Feats(msa_mask=_flat_mask(msa_mask, S * R, msa4.device),
                            pair_mask=_flat_mask(pair_mask, R * R, msa4.device))
        msa, pair, self.saved = eng.block_fwd(0, msa4.reshape(S * R, Cm), pair4.reshape(R * R, Cz), self.feats)
        self.shapes, self.dt = (msa4.shape, pair4.shape), dt
        return msa.view(msa4.shape), pair.view(pair4.shape)

    def bwd(self, g_msa, g_pair):
        (ms, ps) = self.shapes
        dev = self.feats.msa_mask.device
        d_msa = (_f32_copy(g_msa, (ms[1] * ms[2], ms[3])) if g_msa is not None
                 else torch.zeros((ms[1] * ms[2], ms[3]), dtype=F32, device=dev))
        d_pair = (_f32_copy(g_pair, (ps[1] * ps[2], ps[3])) if g_pair is not None
                  else torch.zeros((ps[1] * ps[2], ps[3]), dtype=F32, device=dev))
        # the deferred bias / LN-affine partial rows live for this call only
        self.eng.arena = torch.empty(96 << 20, dtype=torch.uint8, device=dev)
        with self.eng.deferred():
            self.eng.block_bwd(0, d_msa, d_pair, self.saved, self.feats)
        self.eng.arena = None
        self.saved = None
        return (_to_dtype(d_msa, self.dt).view(ms), _to_dtype(d_pair, self.dt).view(ps), None, None,
                *_params_grads(self.store, self.named))


def evoformer_block(state: TrackState, blk: BlockParams, masks: Masks, par=None, policy: ExecPolicy = None,
                    cfg: ModelConfig = None) -> TrackState:
    """src/model.py:431-445: row -> col -> msa transition; OPM(msa_in) into
    pair -> [TriMul out/in] -> tri start -> tri end -> pair transition.  One
    engine call (both branches, fused residuals, fp32 residual-stream
    gradients); with ``policy.row_chunk`` it composes the module functions."""
    _serial(par)
    policy = policy or ExecPolicy()
    if policy.row_chunk and policy.row_chunk < state.msa.shape[1]:
        msa_in = state.msa
        msa = msa_row_attention(msa_in, state.pair, masks.msa, blk, par, policy)
        msa = msa_col_attention(msa, masks.msa_t, blk, par, policy)
        msa = transition(msa, blk.msa_trans)
        pair = _add(state.pair, outer_product_mean(msa_in, masks.msa, blk.opm, par, cfg))
        if blk.tri_mul_out is not None:
            pair = triangle_multiplication(pair, masks.pair, blk.tri_mul_out, True)
            pair = triangle_multiplication(pair, masks.pair, blk.tri_mul_in, False)
        pair = triangle_attention(pair, masks.pair, blk.tri_start, par, policy, ending=False)
        pair = triangle_attention(pair, masks.pair_t, blk.tri_end, par, policy, ending=True)
        pair = transition(pair, blk.pair_trans)
        return TrackState(msa, pair)
    job = _BlockJob(blk)
    msa, pair = _EngineOp.apply(job, _act(state.msa, "msa"), _act(state.pair, "pair"), masks.msa, masks.pair,
                                *[t for _, t in job.named])
    return TrackState(msa, pair)


class _AddJob:
    differentiable = (True,)

    def fwd(self, a, b):
        a, b = a.contiguous(), b.contiguous()
        out = torch.empty_like(a)
        rows = a.numel() // a.shape[-1]
        ops.bias_residual(a.reshape(rows, -1), b.reshape(rows, -1), None, out.view(rows, -1))
        return out

    def bwd(self, g):
        return g, g


def _add(a, b):
    return _EngineOp.apply(_AddJob(), a, b)


class _EmbedJob:
    differentiable = (True, True)

    def __init__(self, mp: ModelParams, recycle: bool):
        self.named = [(n, getattr(mp, a)) for n, a in _EMBED]
        self.recycle = recycle

    def fwd(self, msa_feat, pair_feat, prev_msa, prev_pair, *params):
        _, S, R, Fd = msa_feat.shape
        dt = act_dtype()
        cm, cz = params[0].shape[1], params[2].shape[1]
        self.store = st = _ModuleStore(self.named, dt)
        cfg0 = ModelConfig(n_blocks=0, n_seq=S, n_res=R, c_m=cm, c_z=cz, heads=1, feat_dim=Fd)
        self.eng = eng = _engine(cfg0, st, dt)
        self.feats = _Feats(msa_feat=msa_feat.reshape(S * R, Fd), pair_feat=pair_feat.reshape(R * R, Fd),
                            msa_mask=torch.zeros(S * R, dtype=F32, device=msa_feat.device))
        prev = None
        if self.recycle:
            prev = (prev_msa.detach().reshape(S * R, cm).contiguous(),
                    prev_pair.detach().reshape(R * R, cz).contiguous())
        msa, pair, self.rec = eng.embed_fwd(self.feats, prev)
        self.shapes = ((1, S, R, cm), (1, R, R, cz))
        return msa.view(self.shapes[0]), pair.view(self.shapes[1])

    def bwd(self, g_msa, g_pair):
        (ms, ps) = self.shapes
        dev = self.feats.msa_feat.device
        d_msa = (_f32_copy(g_msa, (ms[1] * ms[2], ms[3])) if g_msa is not None
                 else torch.zeros((ms[1] * ms[2], ms[3]), dtype=F32, device=dev))
        d_pair = (_f32_copy(g_pair, (ps[1] * ps[2], ps[3])) if g_pair is not None
                  else torch.zeros((ps[1] * ps[2], ps[3]), dtype=F32, device=dev))
        self.eng.embed_bwd(d_msa, d_pair, self.feats, self.rec)
        return (None, None, None, None, *_params_grads(self.store, self.named))


def embed(feats: Features, mp: ModelParams, par=None, prev: TrackState = None, device=None) -> TrackState:
    """src/model.py:448-465: feature projections (+ recycled LayerNorms of the
    previous pass's first MSA row and pair, which carry no gradient)."""
    _serial(par)
    dev = device or mp.msa_embed_w.device

    def up(a):
        return a.to(dev, F32) if isinstance(a, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(a, np.float32)).to(dev)
    mf, pf = up(feats.msa_feat), up(feats.pair_feat)
    job = _EmbedJob(mp, prev is not None)
    msa, pair = _EngineOp.apply(job, mf, pf, None if prev is None else prev.msa,
                                None if prev is None else prev.pair, *[t for _, t in job.named])
    return TrackState(msa, pair)


def model_forward(cfg: ModelConfig, mp: ModelParams, feats: Features, par=None, policy: ExecPolicy = None,
                  prev: TrackState = None) -> TrackState:
    """src/model.py:468-472."""
    _serial(par)
    masks = make_masks(feats, par, device=mp.msa_embed_w.device)
    state = embed(feats, mp, par, prev)
    for blk in mp.blocks:
        state = evoformer_block(state, blk, masks, par, policy, cfg)
    return state


class _LossJob:
    differentiable = (True,)

    def fwd(self, msa, pair):
        msa, pair = msa.contiguous(), pair.contiguous()
        km = float(np.float32(1.0 / msa.numel()))
        kz = float(np.float32(1.0 / pair.numel()))
        loss, self.dm, self.dz = ops.sq_loss(msa.reshape(-1, msa.shape[-1]), pair.reshape(-1, pair.shape[-1]),
                                              km, kz)
        self.shapes, self.dt = (msa.shape, pair.shape), msa.dtype
        return loss.view(())

    def bwd(self, g):
        s = float(g.item()) if g is not None else 1.0
        dm, dz = self.dm, self.dz
        if s != 1.0:
            ops.scale_(dm, s)
            ops.scale_(dz, s)
        return (_to_dtype(dm, self.dt).view(self.shapes[0]), _to_dtype(dz, self.dt).view(self.shapes[1]))


def model_loss(state: TrackState):
    """src/model.py:475-478: mean(msa^2) + mean(pair^2) (one kernel, the
    gradient formed in the same pass)."""
    return _EngineOp.apply(_LossJob(), _act(state.msa, "msa"), _act(state.pair, "pair"))
