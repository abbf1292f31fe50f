"""Evoformer block engine: forward and hand-written backward per module,
on the sm_100a kernels.

Mirrors the reference block (src/model.py:300-445) module by module; the
backward of each module is written out the way the reference's fused-op
closure is (src/attention.py:178-221) instead of going through a tape.
Parameter gradients are written straight into the pooled grad region of
the ``FusionEngine`` (tensor fusion, src/fusion.py) -- nothing is copied.

Data layout in HBM (B=1 as in the reference features):
  msa  [S*R, c_m]   token (s, r) -> row s*R + r      (storage dtype)
  pair [R*R, c_z]   token (i, j) -> row i*R + j      (storage dtype)
  residual-stream gradients d_msa / d_pair: same shapes, fp32
The four attention variants read the same token-major buffers through
(batch, position) strides, so MSA-column and triangle-ending attention need
no transposes (the reference transposes, src/model.py:335-340, 388-397).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .fusion import FusionEngine
from .model import ModelConfig

F32 = torch.float32


@dataclass
class Variant:
    """Attention geometry: problems are (batch b, position l); token row of
    (b, l) is b*sb + l*sl; mask element is mask[b*msb + l*msl]."""

    name: str
    B: int
    L: int
    sb: int
    sl: int
    msb: int
    msl: int
    mask: str          # "msa" or "pair"
    bias: bool         # pair-derived bias present
    swap_xy: bool      # nb[h, i, j] = P[j, i, h] (triangle end) instead of P[i, j, h]
    moff: int = 0      # mask element offset (a DAP shard's first row / column)
    ni: int = 0        # bias source extent [ni, nj] (0: the square n_res x n_res pair)
    nj: int = 0


def variants(cfg: ModelConfig) -> dict:
    S, R = cfg.n_seq, cfg.n_res
    return {
        # src/model.py:320-328: batch s, keys r, mask msa[s, r]
        "row_attn": Variant("row_attn", S, R, R, 1, R, 1, "msa", True, False),
        # src/model.py:331-341: batch r, keys s, mask msa_t[r, s] = msa[s, r]
        "col_attn": Variant("col_attn", R, S, 1, R, 1, R, "msa", False, False),
        # src/model.py:381-398 (start): batch i, keys j, mask pair[i, j]
        "tri_start": Variant("tri_start", R, R, R, 1, R, 1, "pair", True, False),
        # (end): batch j of pair^T, keys i: token (a, b) = pair row b*R + a
        "tri_end": Variant("tri_end", R, R, 1, R, 1, R, "pair", True, True),
    }


class DeviceFeatures:
    """Features resident in HBM (fp32): msa_feat [S*R, F], pair_feat [R*R, F],
    msa_mask [S*R], pair_mask [R*R]."""

    def __init__(self, feats, device, cfg: ModelConfig):
        S, R, F = cfg.n_seq, cfg.n_res, cfg.feat_dim

        def up(a, shape):
            return torch.as_tensor(np.ascontiguousarray(a, np.float32)).reshape(shape).to(device)

        self.msa_feat = up(feats.msa_feat, (S * R, F))
        self.pair_feat = up(feats.pair_feat, (R * R, F))
        self.msa_mask = up(feats.msa_mask, (S * R,))
        self.pair_mask = up(feats.pair_mask, (R * R,))

    def copy_from_host(self, host):
        """In-place refresh from pinned host tensors (keeps device pointers
        stable for CUDA-graph replay)."""
        for k in ("msa_feat", "pair_feat", "msa_mask", "pair_mask"):
            getattr(self, k).copy_(getattr(host, k), non_blocking=True)


class BlockEngine:
    def __init__(self, cfg: ModelConfig, store: FusionEngine, act_dtype=torch.bfloat16,
                 arena_mb: int = 96):
        cfg.validate()
        self.cfg = cfg
        self.st = store
        self.dt = act_dtype
        self.var = variants(cfg)
        # this worker's shard: sequences s0.., residue rows r0..r0+r_loc (whole model here)
        self.s0, self.r0, self.r_loc = 0, 0, cfg.n_res
        self.opm_num_dtype = act_dtype
        self._rec = None
        # MSA branch on a second stream (EVO_BRANCH_STREAMS=0 disables)
        import os
        self.branch_streams = (torch.device(store.device).type == "cuda"
                               and os.environ.get("EVO_BRANCH_STREAMS", "1") != "0")
        self._s2 = None
        self.opm_dnum_fused = os.environ.get("EVO_OPM_DNUM_TC", "1") != "0"
        # d(LN output) from the dX GEMMs in the activation dtype: the bf16 policy
        # stores it in bf16 like every other GEMM operand / output of the
        # backward (EVO_DXL_BF16=0 keeps fp32); the LayerNorm backward upcasts
        self._dy_dt = act_dtype if os.environ.get("EVO_DXL_BF16", "1") != "0" else torch.float32
        # triangle attention: input LayerNorm + pair bias in one pass (EVO_LN_PB=0: two ops)
        self.ln_pb_fused = act_dtype == torch.bfloat16 and os.environ.get("EVO_LN_PB", "1") != "0"
        # partial rows of the deferred bias / LN-affine reductions of one block backward
        self.arena = torch.empty(arena_mb << 20, dtype=torch.uint8, device=store.device)
        # two arenas for the block-pipelined backward (blocks_bwd), alternating by block
        self.arenas = (self.arena, torch.empty(arena_mb << 20, dtype=torch.uint8, device=store.device))
        # merged Q|K|V|G projection weights [C, 4*H*c] per attention module (the
        # reference concatenates Wq|Wk|Wv the same way, src/attention.py:133-141),
        # refreshed from the (bf16 shadow of the) pooled params every step
        self.wcat = {}
        srcs, dsts, Cs, Ns = [], [], [], []
        for i in range(cfg.n_blocks):
            for mod, C in (("row_attn", cfg.c_m), ("col_attn", cfg.c_m), ("tri_start", cfg.c_z),
                           ("tri_end", cfg.c_z)):
                p = f"block{i}.{mod}"
                buf = torch.empty((C, 4 * C), dtype=act_dtype, device=store.device)
                self.wcat[p] = buf
                srcs += [store.weight(f"{p}.attn.{f}") for f in ("wq", "wk", "wv", "wg")]
                dsts.append(buf)
                Cs.append(C)
                Ns.append(C)
        if cfg.trimul:  # [ap | ag | bp | bg] projections of TriangleMultiplication
            ch = cfg.c_hidden_mul
            for i in range(cfg.n_blocks):
                for mod in ("tri_mul_out", "tri_mul_in"):
                    p = f"block{i}.{mod}"
                    buf = torch.empty((cfg.c_z, 4 * ch), dtype=act_dtype, device=store.device)
                    self.wcat[p] = buf
                    srcs += [store.weight(f"{p}.w_{nm}") for nm in ("ap", "ag", "bp", "bg")]
                    dsts.append(buf)
                    Cs.append(cfg.c_z)
                    Ns.append(ch)
        wdt = ops.dcode(store.weight(f"block0.row_attn.attn.wq")) if cfg.n_blocks else 0
        adt = ops.dcode(torch.empty(0, dtype=act_dtype))
        self._pack = ops.PackPlan(srcs, dsts, Cs, Ns, False, wdt, adt)
        # merged [w_left | w_right] OPM projection [c_m, 2k]: one GEMM each way
        srcs, dsts = [], []
        for i in range(cfg.n_blocks):
            p = f"block{i}.opm"
            self.wcat[p] = torch.empty((cfg.c_m, 2 * cfg.opm_dim), dtype=act_dtype, device=store.device)
            srcs += [store.weight(f"{p}.w_left"), store.weight(f"{p}.w_right")]
            dsts.append(self.wcat[p])
        self._pack_opm = ops.PackPlan(srcs, dsts, [cfg.c_m] * cfg.n_blocks, [cfg.opm_dim] * cfg.n_blocks,
                                      False, wdt, adt, ns=2)
        self.refresh_weights()

    def refresh_weights(self):
        """Re-pack the merged projection weights after an optimizer step."""
        if self._pack.n:
            self._pack.run()
        if self._pack_opm.n:
            self._pack_opm.run()

    def deferred(self):
        """Batch the ~40 small parameter-gradient reductions of a block backward
        into one finalisation launch."""
        return ops.deferred_reductions(self.arena)

    # -- parameter access ---------------------------------------------------------

    def P(self, name):
        return self.st.param(name)

    def G(self, name):
        return self.st.grad(name)

    def W(self, name, rows):
        """Projection weight in the storage dtype as a [rows, cols] matrix."""
        w = self.st.weight(name)
        return w.view(rows, -1)

    def Gm(self, name, rows):
        return self.st.grad(name).view(rows, -1)

    def mask(self, feats: DeviceFeatures, which: str):
        return feats.msa_mask if which == "msa" else feats.pair_mask

    def _rec_for(self, feats: DeviceFeatures):
        """The OPM normaliser rec = 1/(mask^T mask + 1e-3) of this worker's rows:
        a function of the MSA mask only, so it is computed once per forward pass
        (``embed_fwd`` drops the previous one) and shared by every block."""
        if self._rec is None:
            self._rec = ops.opm_rec(feats.msa_mask, self.cfg.n_seq, self.cfg.n_res, self.r0, self.r_loc)
        return self._rec

    # -- sharding hooks: identities here, collectives in the DAP engine (dap.py) ----

    def _gather_bias(self, nb, v: Variant):
        return nb

    def _scatter_dbias(self, dnb, v: Variant):
        return dnb

    def _opm_reduce(self, num):
        return num

    def _opm_gather(self, dnum):
        return dnum

    def _feat_rows(self, feats: DeviceFeatures):
        """(msa_feat, pair_feat, msa_mask) rows of this worker's shard."""
        return feats.msa_feat, feats.pair_feat, feats.msa_mask

    def _ln_bwd_chain(self, x, dxl, mu, rs, prefix, d, nxt):
        """LayerNorm backward into the residual gradient d (in place).  With
        ``nxt`` (the output-bias gradient slot of the module that runs next in
        the backward) it also returns that module's bf16 operand d_act and
        writes the bias gradient, so the module skips its colsum/cast pass."""
        if nxt is None or self.dt != torch.bfloat16:
            ops.layernorm_bwd(x, dxl, mu, rs, self.P(f"{prefix}.ln_g"), d, d, self.G(f"{prefix}.ln_g"),
                              self.G(f"{prefix}.ln_b"))
            return None
        d_act = torch.empty(d.shape, dtype=self.dt, device=d.device)
        ops.layernorm_bwd_ex(x, dxl, mu, rs, self.P(f"{prefix}.ln_g"), d, d, self.G(f"{prefix}.ln_g"),
                             self.G(f"{prefix}.ln_b"), d_act, nxt)
        return d_act

    # -- gated attention module (LN -> [pair bias] -> fused attention -> residual)

    def attn_fwd(self, x, prefix, v: Variant, feats, pair=None):
        cfg, dt = self.cfg, self.dt
        T, C = x.shape
        H = cfg.heads
        D = C // H
        HD = H * D
        fused = None
        if v.bias and pair is None and self.ln_pb_fused:
            # triangle attention: its LayerNorm and its pair-bias LayerNorm read the
            # same rows -- one pass (csrc/pair_bias_mma.cu), shared statistics
            fused = ops.ln_pair_bias_fwd(x, self.P(f"{prefix}.ln_g"), self.P(f"{prefix}.ln_b"),
                                         self.P(f"{prefix}.bias_ln_g"), self.P(f"{prefix}.bias_ln_b"),
                                         self.P(f"{prefix}.w_bias"), cfg.n_res, H, v.swap_xy,
                                         ni=v.ni or None, nj=v.nj or None)
        nb = pmu = prs = None
        if fused is not None:
            xl, nb, mu, rs = fused
            pmu, prs = mu, rs
            nb = self._gather_bias(nb, v)
        else:
            xl, mu, rs = ops.layernorm(x, self.P(f"{prefix}.ln_g"), self.P(f"{prefix}.ln_b"), dt)
        if v.bias and fused is None:
            z = pair if pair is not None else x
            nb, pmu, prs = ops.pair_bias_fwd(z, self.P(f"{prefix}.bias_ln_g"),
                                             self.P(f"{prefix}.bias_ln_b"),
                                             self.P(f"{prefix}.w_bias"), cfg.n_res, H, v.swap_xy,
                                             ni=v.ni or None, nj=v.nj or None)
            nb = self._gather_bias(nb, v)
        qkvg = torch.empty((T, 4 * HD), dtype=dt, device=x.device)
        ops.gemm(xl, self.wcat[prefix], qkvg)                         # one merged projection
        mask = self.mask(feats, v.mask)[v.moff:]
        ctx, gate, gated, lse = ops.attn_fwd(qkvg, mask, v.msb, v.msl, nb,
                                             self.P(f"{prefix}.attn.bg"), v.B, v.L, H, D, v.sb, v.sl)
        out = torch.empty((T, C), dtype=dt, device=x.device)
        ops.gemm_bias(gated, self.W(f"{prefix}.attn.wo", HD), out, self.P(f"{prefix}.attn.bo"), res=x,
                      bias16=self.st.weight(f"{prefix}.attn.bo"))
        saved = dict(x=x, xl=xl, mu=mu, rs=rs, qkvg=qkvg, ctx=ctx, gate=gate, gated=gated, lse=lse,
                     nb=nb, pmu=pmu, prs=prs, pair=pair if pair is not None else x)
        return out, saved

    def attn_bwd(self, d, sv, prefix, v: Variant, feats, dpair=None, d_act=None, nxt=None, late=None):
        """``d`` (fp32 [T, C]) is d(out) on entry and d(x) on exit.  The
        pair-bias gradient is added into ``dpair`` (or ``d`` for triangle
        attention, whose bias comes from its own input).  ``d_act``: bf16 d(out)
        with the output-bias gradient already taken (from the previous LN
        backward); returns the next module's d_act when ``nxt`` is given."""
        cfg, dt = self.cfg, self.dt
        T, C = d.shape
        H = cfg.heads
        D = C // H
        HD = H * D
        if d_act is None:
            d_act = torch.empty((T, C), dtype=dt, device=d.device)
            ops.colsum_cast(d, self.G(f"{prefix}.attn.bo"), y=d_act)
        ops.gemm(sv["gated"], d_act, self.Gm(f"{prefix}.attn.wo", HD), ta=True)
        dgated = torch.empty((T, HD), dtype=dt, device=d.device)
        ops.gemm(d_act, self.W(f"{prefix}.attn.wo", HD), dgated, tb=True)
        del d_act
        mask = self.mask(feats, v.mask)[v.moff:]
        dqkvg, dnb = ops.attn_bwd(sv["qkvg"], mask, v.msb, v.msl, sv["nb"], sv["ctx"], sv["gate"],
                                  dgated, sv["lse"], self.G(f"{prefix}.attn.bg"), v.B, v.L, H, D,
                                  v.sb, v.sl, want_dbias=v.bias)
        del dgated
        if v.bias:
            dnb = self._scatter_dbias(dnb, v)
        xl = sv["xl"]
        dwcat = torch.empty((C, 4 * HD), dtype=F32, device=d.device)
        ops.gemm(xl, dqkvg, dwcat, ta=True)                           # d[Wq|Wk|Wv|Wg] in one GEMM
        ops.PackPlan([dwcat], [self.Gm(f"{prefix}.attn.{f}", C) for f in ("wq", "wk", "wv", "wg")],
                     [C], [HD], True, ops.F32, ops.F32).run()
        dxl = torch.empty((T, C), dtype=self._dy_dt, device=d.device)
        ops.gemm(dqkvg, self.wcat[prefix], dxl, tb=True)
        del dqkvg, dwcat
        if v.bias:
            target = dpair if dpair is not None else d

            def pair_bias_bwd(dz16=None, dzsum=None):
                # dz16 / dzsum: when the caller knows this is the last write to the
                # pair gradient, the next module's bf16 operand and b2 gradient
                ops.pair_bias_bwd(sv["pair"], sv["pmu"], sv["prs"], self.P(f"{prefix}.bias_ln_g"),
                                  self.P(f"{prefix}.bias_ln_b"), self.P(f"{prefix}.w_bias"), dnb,
                                  v.swap_xy, target, self.G(f"{prefix}.bias_ln_g"),
                                  self.G(f"{prefix}.bias_ln_b"), self.G(f"{prefix}.w_bias"),
                                  cfg.n_res, H, ni=v.ni or None, nj=v.nj or None, dz16=dz16, dzsum=dzsum)
            if dpair is not None and late is not None:
                late.append(pair_bias_bwd)  # into the pair gradient: run by the caller after its join
            else:
                pair_bias_bwd()  # before the LN backward, so d is final when that pass reads it
        return self._ln_bwd_chain(sv["x"], dxl, sv["mu"], sv["rs"], prefix, d, nxt)

    # -- transition (src/model.py:344-348) ------------------------------------------

    def trans_fwd(self, x, prefix):
        dt = self.dt
        T, C = x.shape
        xl, mu, rs = ops.layernorm(x, self.P(f"{prefix}.ln_g"), self.P(f"{prefix}.ln_b"), dt)
        w1 = self.W(f"{prefix}.w1", C)
        h = torch.empty((T, w1.shape[1]), dtype=dt, device=x.device)
        ops.gemm_bias(xl, w1, h, self.P(f"{prefix}.b1"), relu=True, bias16=self.st.weight(f"{prefix}.b1"))
        out = torch.empty((T, C), dtype=dt, device=x.device)
        ops.gemm_bias(h, self.W(f"{prefix}.w2", w1.shape[1]), out, self.P(f"{prefix}.b2"), res=x,
                      bias16=self.st.weight(f"{prefix}.b2"))
        return out, dict(x=x, xl=xl, mu=mu, rs=rs, h=h)

    def trans_bwd(self, d, sv, prefix, nxt=None, d_act=None):
        """``d_act``: bf16 d(out) with the b2 gradient already taken (emitted by
        the LayerNorm backward that last wrote ``d``)."""
        dt = self.dt
        T, C = d.shape
        h = sv["h"]
        F = h.shape[1]
        if d_act is None:
            d_act = torch.empty((T, C), dtype=dt, device=d.device)
            ops.colsum_cast(d, self.G(f"{prefix}.b2"), y=d_act)
        ops.gemm(h, d_act, self.Gm(f"{prefix}.w2", F), ta=True)
        dh = torch.empty((T, F), dtype=dt, device=d.device)
        if dt == torch.bfloat16:  # ReLU mask and the b1 column sums in the GEMM epilogue
            ops.gemm_relu_mask(d_act, self.W(f"{prefix}.w2", F), h, dh, tb=True, colsum=self.G(f"{prefix}.b1"))
        else:
            ops.gemm(d_act, self.W(f"{prefix}.w2", F), dh, tb=True)
            ops.relu_bwd_colsum_(dh, h, self.G(f"{prefix}.b1"))
        del d_act
        ops.gemm(sv["xl"], dh, self.Gm(f"{prefix}.w1", C), ta=True)
        dxl = torch.empty((T, C), dtype=self._dy_dt, device=d.device)
        ops.gemm(dh, self.W(f"{prefix}.w1", C), dxl, tb=True)
        del dh
        return self._ln_bwd_chain(sv["x"], dxl, sv["mu"], sv["rs"], prefix, d, nxt)

    # -- outer product mean (src/model.py:351-378) -----------------------------------

    def opm_fwd(self, msa_in, prefix, feats, pair_res=None, out=None):
        """Returns pair_res + OPM(msa_in) (or OPM alone when pair_res is None),
        written into ``out`` when given."""
        cfg, dt = self.cfg, self.dt
        S, R, k = cfg.n_seq, cfg.n_res, cfg.opm_dim
        SR, Cm = msa_in.shape
        s_loc, r_loc = SR // R, self.r_loc
        xl, mu, rs = ops.layernorm(msa_in, self.P(f"{prefix}.ln_g"), self.P(f"{prefix}.ln_b"), dt)
        ab = torch.empty((SR, 2 * k), dtype=dt, device=msa_in.device)
        ops.gemm(xl, self.wcat[prefix], ab)                           # [a | c] projections in one GEMM
        a, c = ops.opm_proj(ab, self.P(f"{prefix}.b_left"), self.P(f"{prefix}.b_right"),
                            self._feat_rows(feats)[2], k)
        del ab
        rec = self._rec_for(feats)
        outn = None
        if self.opm_dnum_fused and self.r_loc == R:  # unsharded: sum + normalise + re-layout in one kernel
            outn = ops.opm_outn(a.view(s_loc, R * k), c.view(s_loc, R * k), rec, s_loc, R, k)
        if outn is None:
            num = torch.empty((R * k, R * k), dtype=self.opm_num_dtype, device=msa_in.device)
            ops.gemm(a.view(s_loc, R * k), c.view(s_loc, R * k), num, ta=True)
            num = self._opm_reduce(num)            # the shard's rows of the sum over all sequences
            rec, outn = ops.opm_norm_fwd(num, feats.msa_mask, S, R, k, dt, i0=self.r0, ni=r_loc, rec=rec)
            del num
        if out is None:
            out = torch.empty((r_loc * R, cfg.c_z), dtype=dt, device=msa_in.device)
        ops.gemm_bias(outn, self.W(f"{prefix}.w_out", k * k), out, self.P(f"{prefix}.b_out"), res=pair_res,
                      bias16=self.st.weight(f"{prefix}.b_out"))
        return out, dict(x=msa_in, xl=xl, mu=mu, rs=rs, a=a, c=c, rec=rec, outn=outn)

    def opm_bwd_core(self, d, sv, prefix, feats, d_act=None):
        """d(pair_mid) (fp32) -> dxl (fp32 [S*R, c_m]); the LayerNorm backward is
        applied later by opm_ln_bwd so it can accumulate into d(msa_in).  With
        ``d_act`` (bf16 d(pair_mid), b_out gradient already taken) ``d`` is not read."""
        cfg, dt = self.cfg, self.dt
        S, R, k = cfg.n_seq, cfg.n_res, cfg.opm_dim
        RR, Cz = (d if d is not None else d_act).shape
        SR, Cm = sv["x"].shape
        dev = sv["x"].device
        if d_act is None:
            d_act = torch.empty((RR, Cz), dtype=dt, device=dev)
            ops.colsum_cast(d, self.G(f"{prefix}.b_out"), y=d_act)
        ops.gemm(sv["outn"], d_act, self.Gm(f"{prefix}.w_out", k * k), ta=True)
        dnum = None
        if self.opm_dnum_fused:  # one tcgen05 GEMM with the re-layout in its epilogue (opt-in)
            dnum = ops.opm_dnum(d_act, self.W(f"{prefix}.w_out", k * k), sv["rec"], R, k, ni=self.r_loc)
        if dnum is None:
            doutn = torch.empty((RR, k * k), dtype=dt, device=dev)
            ops.gemm(d_act, self.W(f"{prefix}.w_out", k * k), doutn, tb=True)
            dnum = ops.opm_norm_bwd(doutn, sv["rec"], R, k, dt, ni=self.r_loc)
            del doutn
        del d_act
        dnum = self._opm_gather(dnum)
        s_loc = SR // R
        a2, c2 = sv["a"].view(s_loc, R * k), sv["c"].view(s_loc, R * k)
        da = torch.empty((s_loc, R * k), dtype=dt, device=dev)
        dc = torch.empty((s_loc, R * k), dtype=dt, device=dev)
        ops.gemm(c2, dnum, da, tb=True)
        ops.gemm(a2, dnum, dc)
        del dnum
        d_ab = ops.opm_proj_bwd(da, dc, self._feat_rows(feats)[2], self.G(f"{prefix}.b_left"),
                                self.G(f"{prefix}.b_right"), k)
        xl = sv["xl"]
        dwlr = torch.empty((Cm, 2 * k), dtype=F32, device=dev)
        ops.gemm(xl, d_ab, dwlr, ta=True)                             # d[w_left | w_right] in one GEMM
        ops.PackPlan([dwlr], [self.Gm(f"{prefix}.w_left", Cm), self.Gm(f"{prefix}.w_right", Cm)],
                     [Cm], [k], True, ops.F32, ops.F32, ns=2).run()
        dxl = torch.empty((SR, Cm), dtype=self._dy_dt, device=dev)
        ops.gemm(d_ab, self.wcat[prefix], dxl, tb=True)
        return dxl

    def opm_ln_bwd(self, dxl, sv, prefix, d_msa, nxt=None):
        """d_msa += LN backward of the OPM input.  With ``nxt`` (the b2 slot of
        the MSA transition that runs next in the backward) it also returns
        that module's bf16 operand, bias gradient taken (bf16 only)."""
        if nxt is None or self.dt != torch.bfloat16:
            ops.layernorm_bwd(sv["x"], dxl, sv["mu"], sv["rs"], self.P(f"{prefix}.ln_g"), d_msa, d_msa,
                              self.G(f"{prefix}.ln_g"), self.G(f"{prefix}.ln_b"))
            return None
        d_act = torch.empty(d_msa.shape, dtype=self.dt, device=d_msa.device)
        ops.layernorm_bwd_ex(sv["x"], dxl, sv["mu"], sv["rs"], self.P(f"{prefix}.ln_g"), d_msa, d_msa,
                             self.G(f"{prefix}.ln_g"), self.G(f"{prefix}.ln_b"), d_act, nxt)
        return d_act

    # -- TriangleMultiplication (extension; AF2 Alg 11 outgoing / Alg 12 incoming) ---

    def trimul_fwd(self, x, prefix, feats, outgoing: bool):
        cfg, dt = self.cfg, self.dt
        RR, Cz = x.shape
        R, ch = cfg.n_res, cfg.c_hidden_mul
        P = self.P
        zl, mu, rs = ops.layernorm(x, P(f"{prefix}.ln_in_g"), P(f"{prefix}.ln_in_b"), dt)
        proj = torch.empty((RR, 4 * ch), dtype=dt, device=x.device)
        ops.gemm(zl, self.wcat[prefix], proj)
        gp = torch.empty((RR, Cz), dtype=dt, device=x.device)
        ops.gemm(zl, self.W(f"{prefix}.w_g", Cz), gp)
        biases = [P(f"{prefix}.b_{nm}") for nm in ("ap", "ag", "bp", "bg")]
        a_cm, b_cm = ops.trimul_gate_fwd(proj, biases, feats.pair_mask, ch)
        o_cm = torch.empty((ch, RR), dtype=dt, device=x.device)
        A0, B0, O0 = a_cm[0].view(R, R), b_cm[0].view(R, R), o_cm[0].view(R, R)
        if outgoing:   # o_ij = sum_k a_ik b_jk
            ops.gemm_batched(A0, B0, O0, ch, RR, RR, RR, tb=True)
        else:          # o_ij = sum_k a_ki b_kj
            ops.gemm_batched(A0, B0, O0, ch, RR, RR, RR, ta=True)
        o = ops.transpose2d(o_cm)                                   # [RR, ch]
        del o_cm
        ol, mu2, rs2 = ops.layernorm(o, P(f"{prefix}.ln_out_g"), P(f"{prefix}.ln_out_b"), dt)
        y = torch.empty((RR, Cz), dtype=dt, device=x.device)
        ops.gemm(ol, self.W(f"{prefix}.w_o", ch), y)
        g, out = ops.gated_residual(x, gp, P(f"{prefix}.b_g"), y, P(f"{prefix}.b_o"))
        return out, dict(x=x, zl=zl, mu=mu, rs=rs, proj=proj, a=a_cm, b=b_cm, o=o, mu2=mu2, rs2=rs2,
                         ol=ol, y=y, g=g, outgoing=outgoing)

    def trimul_bwd(self, d, sv, prefix, feats):
        cfg, dt = self.cfg, self.dt
        RR, Cz = d.shape
        R, ch = cfg.n_res, cfg.c_hidden_mul
        P, G = self.P, self.G
        dyb, dgp = ops.gated_residual_bwd(d, sv["g"], sv["y"], P(f"{prefix}.b_o"))
        ops.colsum_cast(dyb, G(f"{prefix}.b_o"))
        ops.colsum_cast(dgp, G(f"{prefix}.b_g"))
        ops.gemm(sv["ol"], dyb, self.Gm(f"{prefix}.w_o", ch), ta=True)
        dol = torch.empty((RR, ch), dtype=self._dy_dt, device=d.device)
        ops.gemm(dyb, self.W(f"{prefix}.w_o", ch), dol, tb=True)
        del dyb
        do = torch.empty((RR, ch), dtype=F32, device=d.device)
        ops.layernorm_bwd(sv["o"], dol, sv["mu2"], sv["rs2"], P(f"{prefix}.ln_out_g"), None, do,
                          G(f"{prefix}.ln_out_g"), G(f"{prefix}.ln_out_b"))
        del dol
        do_cm = ops.transpose2d(do, dt)                              # [ch, RR]
        del do
        a_cm, b_cm = sv["a"], sv["b"]
        da = torch.empty_like(a_cm)
        db = torch.empty_like(b_cm)
        D0, A0, B0 = do_cm[0].view(R, R), a_cm[0].view(R, R), b_cm[0].view(R, R)
        dA0, dB0 = da[0].view(R, R), db[0].view(R, R)
        if sv["outgoing"]:   # o = a b^T: da = do b, db = do^T a
            ops.gemm_batched(D0, B0, dA0, ch, RR, RR, RR)
            ops.gemm_batched(D0, A0, dB0, ch, RR, RR, RR, ta=True)
        else:                # o = a^T b: da = b do^T, db = a do
            ops.gemm_batched(B0, D0, dA0, ch, RR, RR, RR, tb=True)
            ops.gemm_batched(A0, D0, dB0, ch, RR, RR, RR)
        del do_cm
        biases = [P(f"{prefix}.b_{nm}") for nm in ("ap", "ag", "bp", "bg")]
        dproj = ops.trimul_gate_bwd(sv["proj"], biases, feats.pair_mask, da, db, ch)
        del da, db
        # per-slice column sums straight into the grad slots (these may be
        # deferred reductions, so nothing here may read their output)
        for s, nm in enumerate(("ap", "ag", "bp", "bg")):
            ops.colsum_strided(dproj[:, s * ch:(s + 1) * ch], G(f"{prefix}.b_{nm}"), accumulate=True)
        zl = sv["zl"]
        dw4 = torch.empty((Cz, 4 * ch), dtype=F32, device=d.device)
        ops.gemm(zl, dproj, dw4, ta=True)
        ops.PackPlan([dw4], [self.Gm(f"{prefix}.w_{nm}", Cz) for nm in ("ap", "ag", "bp", "bg")],
                     [Cz], [ch], True, ops.F32, ops.F32).run()
        ops.gemm(zl, dgp, self.Gm(f"{prefix}.w_g", Cz), ta=True)
        dzl = torch.empty((RR, Cz), dtype=F32, device=d.device)
        ops.gemm(dproj, self.wcat[prefix], dzl, tb=True)
        ops.gemm(dgp, self.W(f"{prefix}.w_g", Cz), dzl, tb=True, beta=1.0)
        ops.layernorm_bwd(sv["x"], dzl, sv["mu"], sv["rs"], P(f"{prefix}.ln_in_g"), d, d,
                          G(f"{prefix}.ln_in_g"), G(f"{prefix}.ln_in_b"))

    # -- branches (the split used by branch parallelism, src/harness.py:447-486) ----

    def msa_branch_fwd(self, i, msa_in, pair_in, feats):
        p = f"block{i}"
        msa, s1 = self.attn_fwd(msa_in, f"{p}.row_attn", self.var["row_attn"], feats, pair=pair_in)
        msa, s2 = self.attn_fwd(msa, f"{p}.col_attn", self.var["col_attn"], feats)
        msa, s3 = self.trans_fwd(msa, f"{p}.msa_trans")
        return msa, (s1, s2, s3)

    def msa_branch_bwd(self, i, d_msa, d_pair_acc, saved, feats, late=None, d_act=None):
        """d_msa: d(msa_out) -> d(msa_in) in place; the pair-bias path adds
        d(pair_in) into d_pair_acc (appended to ``late`` instead when given).
        ``d_act``: bf16 d_msa with the MSA transition's b2 gradient taken."""
        p = f"block{i}"
        s1, s2, s3 = saved
        a = self.trans_bwd(d_msa, s3, f"{p}.msa_trans", nxt=self.G(f"{p}.col_attn.attn.bo"), d_act=d_act)
        a = self.attn_bwd(d_msa, s2, f"{p}.col_attn", self.var["col_attn"], feats, d_act=a,
                          nxt=self.G(f"{p}.row_attn.attn.bo"))
        self.attn_bwd(d_msa, s1, f"{p}.row_attn", self.var["row_attn"], feats, dpair=d_pair_acc, d_act=a,
                      late=late)

    def pair_branch_fwd(self, i, pair_mid, feats):
        p = f"block{i}"
        pair, tm = pair_mid, []
        if self.cfg.trimul:  # extension, after pair += OPM (SURVEY A14 placement)
            pair, s = self.trimul_fwd(pair, f"{p}.tri_mul_out", feats, True)
            tm.append(s)
            pair, s = self.trimul_fwd(pair, f"{p}.tri_mul_in", feats, False)
            tm.append(s)
        pair, s1 = self.attn_fwd(pair, f"{p}.tri_start", self.var["tri_start"], feats)
        pair, s2 = self.attn_fwd(pair, f"{p}.tri_end", self.var["tri_end"], feats)
        pair, s3 = self.trans_fwd(pair, f"{p}.pair_trans")
        return pair, (tm, s1, s2, s3)

    def pair_branch_bwd(self, i, d_pair, saved, feats, opm_nxt=False, d_act=None):
        """d(pair_out) -> d(pair_mid) in place.  With ``opm_nxt`` (the caller
        runs this block's OPM backward on the same d(pair_mid)) the last
        LayerNorm backward also emits the OPM's bf16 operand and its b_out
        gradient, returned for ``opm_bwd_core(d_act=...)``; else None.
        ``d_act``: bf16 d_pair with the pair transition's b2 gradient taken."""
        p = f"block{i}"
        tm, s1, s2, s3 = saved
        a = self.trans_bwd(d_pair, s3, f"{p}.pair_trans", nxt=self.G(f"{p}.tri_end.attn.bo"), d_act=d_act)
        a = self.attn_bwd(d_pair, s2, f"{p}.tri_end", self.var["tri_end"], feats, d_act=a,
                          nxt=self.G(f"{p}.tri_start.attn.bo"))
        nxt = self.G(f"{p}.opm.b_out") if opm_nxt and not tm else None
        a = self.attn_bwd(d_pair, s1, f"{p}.tri_start", self.var["tri_start"], feats, d_act=a, nxt=nxt)
        if tm:
            self.trimul_bwd(d_pair, tm[1], f"{p}.tri_mul_in", feats)
            self.trimul_bwd(d_pair, tm[0], f"{p}.tri_mul_out", feats)
        return a

    # -- whole block (src/model.py:431-445) -------------------------------------------

    # Branch concurrency on one GPU: given the block inputs, the MSA stack and
    # the OPM + pair stack are independent (the split Branch Parallelism puts on
    # two GPUs, src/harness.py:447-486).  On one GPU the MSA branch runs on a
    # second CUDA stream, forked at the block start and joined at its end, so
    # its kernels fill the SMs the pair branch's kernels leave idle.  Nothing
    # allocated on one stream is freed by the host between fork and join.

    def _side_stream(self):
        if self._s2 is None:
            import os
            prio = int(os.environ.get("EVO_SIDE_PRIORITY", "-1"))  # MSA branch ahead of the pair branch: -0.45 ms per step (A/B)
            self._s2 = torch.cuda.Stream(device=self.st.device, priority=prio)
        return self._s2

    def block_fwd(self, i, msa_in, pair_in, feats):
        if not self.branch_streams:
            msa, sm = self.msa_branch_fwd(i, msa_in, pair_in, feats)
            pair_mid, so = self.opm_fwd(msa_in, f"block{i}.opm", feats, pair_res=pair_in)
            pair, sp = self.pair_branch_fwd(i, pair_mid, feats)
            return msa, pair, (sm, so, sp)
        main, side = torch.cuda.current_stream(), self._side_stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            msa, sm = self.msa_branch_fwd(i, msa_in, pair_in, feats)
        pair_mid, so = self.opm_fwd(msa_in, f"block{i}.opm", feats, pair_res=pair_in)
        pair, sp = self.pair_branch_fwd(i, pair_mid, feats)
        main.wait_stream(side)
        return msa, pair, (sm, so, sp)

    def block_bwd(self, i, d_msa, d_pair, saved, feats):
        """In place: (d msa_out, d pair_out) -> (d msa_in, d pair_in)."""
        sm, so, sp = saved
        if not self.branch_streams:
            a = self.pair_branch_bwd(i, d_pair, sp, feats, opm_nxt=True)  # d_pair = d(pair_mid)
            dxl = self.opm_bwd_core(d_pair, so, f"block{i}.opm", feats, d_act=a)
            self.msa_branch_bwd(i, d_msa, d_pair, sm, feats)      # d_pair += bias path
            self.opm_ln_bwd(dxl, so, f"block{i}.opm", d_msa)      # d_msa += OPM path
            return
        main, side = torch.cuda.current_stream(), self._side_stream()
        late = []
        side.wait_stream(main)
        with torch.cuda.stream(side):
            self.msa_branch_bwd(i, d_msa, d_pair, sm, feats, late=late)
        a = self.pair_branch_bwd(i, d_pair, sp, feats, opm_nxt=True)  # d_pair = d(pair_mid)
        dxl = self.opm_bwd_core(d_pair, so, f"block{i}.opm", feats, d_act=a)
        main.wait_stream(side)
        for fn in late:                                           # d_pair += bias path
            fn()
        self.opm_ln_bwd(dxl, so, f"block{i}.opm", d_msa)          # d_msa += OPM path

    # -- embedding, recycling, loss (src/model.py:448-478, src/harness.py:313-320) ----

    def embed_fwd(self, feats: DeviceFeatures, prev=None):
        cfg, dt = self.cfg, self.dt
        R = cfg.n_res
        mf, pf, _ = self._feat_rows(feats)
        dev = mf.device
        self._rec = None  # the step's mask may have changed: recompute the OPM normaliser
        ym = torch.empty((mf.shape[0], cfg.c_m), dtype=F32, device=dev)
        ops.gemm(mf, self.P("msa_embed.w"), ym)
        msa = torch.empty((mf.shape[0], cfg.c_m), dtype=dt, device=dev)
        ops.bias_residual(None, ym, self.P("msa_embed.b"), msa)
        yz = torch.empty((pf.shape[0], cfg.c_z), dtype=F32, device=dev)
        ops.gemm(pf, self.P("pair_embed.w"), yz)
        pair = torch.empty((pf.shape[0], cfg.c_z), dtype=dt, device=dev)
        ops.bias_residual(None, yz, self.P("pair_embed.b"), pair)
        rec = None
        if prev is not None:
            pm = m1 = r1 = None
            if self.s0 == 0:  # the recycled first MSA row lives on the shard holding sequence 0
                pm = prev[0][:R].contiguous()
                fb, m1, r1 = ops.layernorm(pm, self.P("recycle_m.g"), self.P("recycle_m.b"), F32)
                ops.bias_residual(msa[:R], fb, None, msa[:R])
            pz = prev[1]
            fz, m2, r2 = ops.layernorm(pz, self.P("recycle_z.g"), self.P("recycle_z.b"), F32)
            ops.bias_residual(pair, fz, None, pair)
            rec = (pm, m1, r1, pz, m2, r2)
        return msa, pair, rec

    def embed_bwd(self, d_msa, d_pair, feats: DeviceFeatures, rec, which: str = "both"):
        """``which`` = 'msa' / 'pair' closes out one branch only (BP ranks)."""
        mf, pf, _ = self._feat_rows(feats)
        if which in ("both", "msa"):
            ops.gemm(mf, d_msa, self.G("msa_embed.w"), ta=True)
            ops.colsum_cast(d_msa, self.G("msa_embed.b"))
        if which in ("both", "pair"):
            ops.gemm(pf, d_pair, self.G("pair_embed.w"), ta=True)
            ops.colsum_cast(d_pair, self.G("pair_embed.b"))
        if rec is not None:
            R = self.cfg.n_res
            pm, m1, r1, pz, m2, r2 = rec
            if which in ("both", "msa") and pm is not None:
                scratch = torch.empty_like(d_msa[:R])
                ops.layernorm_bwd(pm, d_msa[:R], m1, r1, self.P("recycle_m.g"), None, scratch,
                                  self.G("recycle_m.g"), self.G("recycle_m.b"))
            if which in ("both", "pair"):
                scratch = torch.empty_like(d_pair)
                ops.layernorm_bwd(pz, d_pair, m2, r2, self.P("recycle_z.g"), None, scratch,
                                  self.G("recycle_z.g"), self.G("recycle_z.b"))

    # -- small helpers used by the parallel step (parallel.py) ---------------------

    def zero_grads(self):
        self.st.zero_grads()

    def grad_region(self):
        return self.st.regions["grads"]

    def block_grad_view(self, i):
        """(view, lo, hi): block i's contiguous slice of the pooled grad region
        (its parameters are consecutive in the flatten order), in elements."""
        spans = getattr(self, "_block_spans", None)
        if spans is None:
            spans = {}
            for sl in self.st.slots:
                if sl.name.startswith("block"):
                    b = int(sl.name.split(".")[0][5:])
                    lo, hi = sl.offset // 4, (sl.offset + sl.padded_bytes) // 4
                    cur = spans.get(b)
                    spans[b] = (lo, hi) if cur is None else (min(cur[0], lo), max(cur[1], hi))
            self._block_spans = spans
        lo, hi = spans[i]
        return self.grad_region()[lo:hi], lo, hi

    def empty_like(self, t):
        return torch.empty_like(t)

    def zeros_like(self, t):
        return torch.zeros_like(t)

    def add(self, a, b):
        out = torch.empty_like(a)
        ops.bias_residual(a, b, None, out)
        return out

    def loss(self, msa, pair):
        cfg = self.cfg
        km = float(np.float32(1.0 / (cfg.n_seq * cfg.n_res * cfg.c_m)))
        kz = float(np.float32(1.0 / (cfg.n_res * cfg.n_res * cfg.c_z)))
        return ops.sq_loss(msa, pair, km, kz)

    # -- whole model ---------------------------------------------------------------------

    def blocks_fwd(self, msa, pair, feats, saved=None, inputs=None):
        """All blocks forward; appends each block's saved tensors to ``saved``
        and, for recompute, each block's (msa, pair) input to ``inputs``.

        With branch streams the OPM of block i+1 (which needs only block i's
        MSA output) is computed on the side stream right after block i's MSA
        branch, i.e. while the main stream runs block i's pair branch; the main
        stream then only adds it onto the pair activations (event-ordered).  Its
        output buffers are allocated on the main stream, which consumes them."""
        n = self.cfg.n_blocks
        if not self.branch_streams or n == 0:
            for i in range(n):
                if inputs is not None:
                    inputs.append((msa, pair))
                msa, pair, sv = self.block_fwd(i, msa, pair, feats)
                if saved is not None:
                    saved.append(sv)
            return msa, pair
        main, side = torch.cuda.current_stream(), self._side_stream()
        RR, Cz = pair.shape

        def opm_on_side(i, msa_i):
            y = torch.empty((RR, Cz), dtype=self.dt, device=pair.device)  # main-stream allocation
            ev = torch.cuda.Event()
            with torch.cuda.stream(side):
                _, so = self.opm_fwd(msa_i, f"block{i}.opm", feats, pair_res=None, out=y)
                ev.record(side)
            return y, so, ev

        side.wait_stream(main)
        nxt = opm_on_side(0, msa)
        for i in range(n):
            if inputs is not None:
                inputs.append((msa, pair))
            y, so, ev = nxt
            side.wait_stream(main)                   # pair (row-attention bias) is final
            with torch.cuda.stream(side):
                msa_new, sm = self.msa_branch_fwd(i, msa, pair, feats)
            if i + 1 < n:
                nxt = opm_on_side(i + 1, msa_new)
            main.wait_event(ev)                      # OPM(block i) done on the side stream
            pair_mid = torch.empty_like(pair)
            ops.bias_residual(pair, y, None, pair_mid)
            del y
            pair, sp = self.pair_branch_fwd(i, pair_mid, feats)
            msa = msa_new
            if saved is not None:
                saved.append((sm, so, sp))
        main.wait_stream(side)
        return msa, pair

    def block_refwd(self, i, msa_in, pair_in, feats):
        """Recompute block i's saved tensors from its inputs
        (src/trainer.py:108-179 ``recompute_grads``): same kernels, same op
        order and the same stream placement as ``blocks_fwd`` -- the OPM
        output is added onto the pair activations as a separate bf16 tensor
        there, so it is here too -- so the recomputed tensors, and therefore
        the gradients, are bitwise those of the stored-activation pass."""
        if not self.branch_streams:
            return self.block_fwd(i, msa_in, pair_in, feats)[2]
        main, side = torch.cuda.current_stream(), self._side_stream()
        y = torch.empty(pair_in.shape, dtype=self.dt, device=pair_in.device)  # main-stream allocation
        ev = torch.cuda.Event()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            _, so = self.opm_fwd(msa_in, f"block{i}.opm", feats, pair_res=None, out=y)
            ev.record(side)
            _, sm = self.msa_branch_fwd(i, msa_in, pair_in, feats)
        main.wait_event(ev)
        pair_mid = torch.empty_like(pair_in)
        ops.bias_residual(pair_in, y, None, pair_mid)
        del y
        _, sp = self.pair_branch_fwd(i, pair_mid, feats)
        return sm, so, sp

    def blocks_bwd(self, d_msa, d_pair, saved, feats, inputs=None, grad_ready=None):
        """All blocks backward, in place on (d_msa, d_pair); frees ``saved``.

        With ``inputs`` (recompute) ``saved`` is unused: block i's saved tensors are recomputed from ``inputs[i]`` right before its
        backward, so at most one block's activations are alive at a time.

        With branch streams the MSA branch runs on the side stream as in
        ``block_bwd``, and the OPM backward of block i -- which needs only a bf16
        copy of d(pair_mid) -- also moves to the side stream, where it overlaps
        the main stream's pair-branch backward of block i-1.  The per-block
        deferred reductions then alternate between two arenas and are finalised
        on the side stream once both streams' kernels of the block are done.

        ``grad_ready(i, stream)`` is called once block i's parameter gradients
        are final on ``stream`` (None: the current stream) -- the hook of the
        bucketed data-parallel gradient all-reduce (parallel._GradBuckets)."""
        n = self.cfg.n_blocks
        if inputs is not None:
            saved = [None] * n
        if not self.branch_streams:
            for i in reversed(range(n)):
                if inputs is not None:
                    saved[i] = self.block_refwd(i, *inputs[i], feats)
                with self.deferred():
                    self.block_bwd(i, d_msa, d_pair, saved[i], feats)
                if grad_ready is not None:
                    grad_ready(i, None)
                saved[i] = None
            return
        main, side = torch.cuda.current_stream(), self._side_stream()
        keep = []  # main-stream tensors read by the side stream: alive until the final join
        side.wait_stream(main)
        msa_act = None  # block i-1's MSA transition operand, emitted by block i's OPM LN backward
        pair_act = None  # block i-1's pair transition operand, emitted by block i's row-attention pair bias
        for i in reversed(range(n)):
            if inputs is not None:
                saved[i] = self.block_refwd(i, *inputs[i], feats)
            sm, so, sp = saved[i]
            ops.defer_begin(self.arenas[i % 2])
            late = []
            with torch.cuda.stream(side):
                self.msa_branch_bwd(i, d_msa, d_pair, sm, feats, late=late, d_act=msa_act)
                msa_act = None
                ev_msa = torch.cuda.Event()
                ev_msa.record(side)
            d_act = self.pair_branch_bwd(i, d_pair, sp, feats, opm_nxt=True, d_act=pair_act)  # d(pair_mid)
            pair_act = None
            if d_act is None:
                d_act = torch.empty(d_pair.shape, dtype=self.dt, device=d_pair.device)
                ops.colsum_cast(d_pair, self.G(f"block{i}.opm.b_out"), y=d_act)
            ev_pair = torch.cuda.Event()
            ev_pair.record(main)
            main.wait_event(ev_msa)
            for k, fn in enumerate(late):                       # d_pair += bias path
                if k == len(late) - 1 and i > 0 and self.dt == torch.bfloat16:
                    # the last write to d(pair_in): it also emits block i-1's pair
                    # transition operand and b2 gradient
                    pair_act = torch.empty(d_pair.shape, dtype=self.dt, device=d_pair.device)
                    fn(dz16=pair_act, dzsum=self.G(f"block{i - 1}.pair_trans.b2"))
                else:
                    fn()
            with torch.cuda.stream(side):
                side.wait_event(ev_pair)
                dxl = self.opm_bwd_core(None, so, f"block{i}.opm", feats, d_act=d_act)
                msa_act = self.opm_ln_bwd(dxl, so, f"block{i}.opm", d_msa,  # d_msa += OPM path
                                          nxt=self.G(f"block{i - 1}.msa_trans.b2") if i > 0 else None)
                del dxl
                side.wait_stream(main)                          # every partial of block i written
                ops.defer_end(side)
                if grad_ready is not None:
                    grad_ready(i, side)
            keep.append(d_act)
            saved[i] = None
        main.wait_stream(side)
        keep.clear()

    def forward_only(self, feats, prev=None):
        msa, pair, _ = self.embed_fwd(feats, prev)
        return self.blocks_fwd(msa, pair, feats)

    def forward_backward(self, feats: DeviceFeatures, n_cycles: int = 1, recompute: bool = False,
                         grad_ready=None):
        """``_serial_grads`` (src/harness.py:327-352): n-1 untaped recycling
        passes, one differentiated pass; grads land in the pooled region.
        ``recompute`` keeps only each block's inputs through the forward and
        recomputes its activations during the backward
        (src/trainer.py:108-179).  Returns (loss device tensor [1], (msa, pair))."""
        self.refresh_weights()
        self.st.zero_grads()
        prev = None
        for _ in range(max(0, n_cycles - 1)):
            prev = self.forward_only(feats, prev)
        msa, pair, rec = self.embed_fwd(feats, prev)
        if recompute:
            saved, inputs = None, []
            msa, pair = self.blocks_fwd(msa, pair, feats, None, inputs)
        else:
            saved, inputs = [], None
            msa, pair = self.blocks_fwd(msa, pair, feats, saved)
        loss, d_msa, d_pair = self.loss(msa, pair)
        self.blocks_bwd(d_msa, d_pair, saved, feats, inputs, grad_ready=grad_ready)
        if inputs is not None:
            inputs.clear()                       # blocks_bwd joined the side stream
        with self.deferred():
            self.embed_bwd(d_msa, d_pair, feats, rec)
        return loss, (msa, pair)
