"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/gen_goldens.py

It imports ``evotrain`` from ``/root/reference/pkg/src`` and writes small
``.npz`` fixtures next to this script.  The fixtures travel with the repo;
the tests never read ``/root/reference`` at run time.

Fixtures
--------
prng.npz          splitmix64 outputs and uniform draws (src/prng.py:19-53)
attn_ops.npz      gated_attention_fused fwd + grads of mean(o^2) for the
                  reference's own randomized attention cases
                  (tests/test_attention.py:15-27), including head dims 4/8/16/32
                  and a fully-masked row
model_O.npz       one Evoformer block at the oracle shape (S=32, R=64,
                  c_m=64, c_z=32, H=2, opm=32): loss, outputs, every grad
model_O_h4.npz    the same with heads=4 (head dims 16/8)
model_mini.npz    the reference mini config (2 blocks, S=8, R=16, H=4) with
                  n_cycles=2 (exercises recycling)
optim.npz         FusionEngine fused trajectory: 4 steps over 7 params
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from evotrain import harness as H  # noqa: E402
from evotrain import model as M  # noqa: E402
from evotrain import runtime  # noqa: E402
from evotrain import tensor as T  # noqa: E402
from evotrain.attention import (AttentionInput, AttentionParams,  # noqa: E402
                                gated_attention_fused)
from evotrain.autodiff import Tape, backward  # noqa: E402
from evotrain.fusion import FusionEngine, OptimConfig  # noqa: E402
from evotrain.prng import Prng, splitmix64  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def gen_prng():
    seeds = [0, 1, 7, 32, 2**63 + 5]
    out = {}
    for i, s in enumerate(seeds):
        out[f"sm_{i}"] = np.array(splitmix64(s, 16), dtype=np.uint64)
        out[f"seed_{i}"] = np.array(s, dtype=np.uint64)
        r = Prng(s)
        out[f"uni_{i}"] = np.concatenate([r.uniform((3, 5)).ravel(), r.uniform((7,)).ravel()])
    return out


def attn_case(seed, b, s, r, h, c, full_mask_row):
    """Inputs drawn like tests/test_attention.py:15-27."""
    rng = Prng(seed)
    cdim = h * c
    u = lambda *sh: T.parameter(rng.uniform(sh) * 0.2)  # noqa: E731
    p = AttentionParams(u(cdim, h, c), u(cdim, h, c), u(cdim, h, c),
                        u(cdim, h, c), u(h, c), u(h, c, cdim), u(cdim))
    x = T.parameter(rng.uniform((b, s, r, cdim)))
    mask = np.ones((b, s, r), np.float32)
    mask[..., -1] = 0.0
    if full_mask_row:
        mask[:, 0, :] = 0.0
    nb = T.parameter(rng.uniform((h, r, r)) * 0.1)
    return AttentionInput(x, T.tensor(mask), nb), p, x, nb, mask


ATTN_CASES = [
    # seed, b, s, r, h, c, full_mask_row, use_bias
    (0, 1, 3, 5, 2, 4, False, True),
    (1, 1, 4, 8, 2, 8, False, True),
    (2, 1, 2, 16, 4, 16, True, True),
    (3, 1, 3, 24, 2, 32, False, True),
    (4, 1, 5, 12, 2, 16, True, False),
    (5, 1, 2, 33, 3, 32, False, True),
]


def gen_attn():
    out = {}
    for k, (seed, b, s, r, h, c, fm, use_bias) in enumerate(ATTN_CASES):
        runtime.set_context(runtime.Context())
        inp, p, x, nb, mask = attn_case(seed, b, s, r, h, c, fm)
        if not use_bias:
            inp = AttentionInput(inp.x, inp.mask, None)
        params = [x] + ([nb] if use_bias else []) + p.all()
        with Tape() as t:
            o = gated_attention_fused(inp, p)
            loss = T.mean_all(T.mul(o, o))
        g = backward(t, loss, params)
        t.close()
        out[f"c{k}_meta"] = np.array([seed, b, s, r, h, c, int(fm), int(use_bias)])
        out[f"c{k}_x"] = x.data.copy()
        out[f"c{k}_mask"] = mask
        if use_bias:
            out[f"c{k}_nb"] = nb.data.copy()
        for name, t_ in zip(("wq", "wk", "wv", "wg", "bg", "wo", "bo"), p.all()):
            out[f"c{k}_p_{name}"] = t_.data.copy()
        out[f"c{k}_out"] = o.data.copy()
        names = ["x"] + (["nb"] if use_bias else []) + ["wq", "wk", "wv", "wg", "bg", "wo", "bo"]
        for name, pp in zip(names, params):
            out[f"c{k}_g_{name}"] = g[pp.bid].data.copy()
    return out


def gen_model(cfg, n_cycles, feat_seed=3, param_seed=7):
    runtime.set_context(runtime.Context())
    mp = M.init_params(cfg, param_seed)
    feats = M.make_features(cfg, feat_seed)
    loss, grads, (msa, pair) = H._serial_grads(cfg, mp, feats, M.ExecPolicy(), n_cycles)
    out = {"cfg": np.array([cfg.n_blocks, cfg.n_seq, cfg.n_res, cfg.c_m, cfg.c_z,
                            cfg.heads, cfg.opm_dim, n_cycles, feat_seed, param_seed]),
           "loss": np.array(loss, np.float64), "msa": msa, "pair": pair,
           "msa_feat": feats.msa_feat, "pair_feat": feats.pair_feat}
    for n, _ in M.flatten_params(mp):
        out[f"g::{n}"] = grads[n]
    return out


def gen_optim():
    rng = Prng(3)
    params = [(f"p{i}", T.parameter(rng.uniform((3, i + 1)) * 0.1)) for i in range(7)]
    init = {n: t.data.copy() for n, t in params}
    eng = FusionEngine(params, OptimConfig(), fused=True)
    grng = Prng(4)
    out = {}
    for n, v in init.items():
        out[f"init::{n}"] = v
    for step in range(4):
        grads = {n: grng.uniform(t.shape) * (0.5 if step != 2 else 1e-3) for n, t in params}
        for n, g in grads.items():
            out[f"grad{step}::{n}"] = g
        out[f"norm{step}"] = np.array(eng.apply(grads), np.float64)
        for n, t in params:
            out[f"param{step}::{n}"] = t.data.copy()
            out[f"ema{step}::{n}"] = eng.view("ema", n).copy()
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "prng.npz"), **gen_prng())
    np.savez_compressed(os.path.join(HERE, "attn_ops.npz"), **gen_attn())
    cfg_o = M.ModelConfig(n_blocks=1, n_seq=32, n_res=64, c_m=64, c_z=32, heads=2, opm_dim=32)
    np.savez_compressed(os.path.join(HERE, "model_O.npz"), **gen_model(cfg_o, 1))
    cfg_o4 = M.ModelConfig(n_blocks=1, n_seq=32, n_res=64, c_m=64, c_z=32, heads=4, opm_dim=32)
    np.savez_compressed(os.path.join(HERE, "model_O_h4.npz"), **gen_model(cfg_o4, 1))
    cfg_mini = M.ModelConfig(n_blocks=2, n_seq=8, n_res=16, c_m=32, c_z=16, heads=4, opm_dim=4)
    np.savez_compressed(os.path.join(HERE, "model_mini.npz"), **gen_model(cfg_mini, 2))
    np.savez_compressed(os.path.join(HERE, "optim.npz"), **gen_optim())
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
