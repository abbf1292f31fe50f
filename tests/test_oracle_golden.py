"""Pin the CPU oracle (oracle/evoformer_np.py) to golden vectors produced by
the reference package itself (tests/golden/gen_goldens.py)."""

import numpy as np
import pytest

from conftest import load_golden, rel_err
from oracle import evoformer_np as O


def test_prng_bit_exact():
    g = load_golden("prng.npz")
    for i in range(5):
        seed = int(g[f"seed_{i}"])
        assert np.array_equal(np.array(O.splitmix64(seed, 16), np.uint64), g[f"sm_{i}"])
        r = O.Prng(seed)
        got = np.concatenate([r.uniform((3, 5)).ravel(), r.uniform((7,)).ravel()])
        assert np.array_equal(got, g[f"uni_{i}"])


def _attn_case(g, k):
    seed, b, s, r, h, c, fm, use_bias = (int(v) for v in g[f"c{k}_meta"])
    p = {f: g[f"c{k}_p_{f}"] for f in O.ATTN_FIELDS}
    nb = g[f"c{k}_nb"] if use_bias else None
    return g[f"c{k}_x"], g[f"c{k}_mask"], nb, p


@pytest.mark.parametrize("k", range(6))
def test_attention_matches_reference(k):
    g = load_golden("attn_ops.npz")
    x, mask, nb, p = _attn_case(g, k)
    out, cache = O.attention_fwd(x, mask, nb, p)
    assert rel_err(out, g[f"c{k}_out"]) <= 1e-6
    dout = (2.0 / out.size) * out  # d mean(o^2)
    dx, dp, dnb = O.attention_bwd(dout.astype(np.float32), cache)
    assert rel_err(dx, g[f"c{k}_g_x"]) <= 1e-5
    for f in O.ATTN_FIELDS:
        assert rel_err(dp[f], g[f"c{k}_g_{f}"], 1e-8) <= 1e-5, f
    if nb is not None:
        assert rel_err(dnb, g[f"c{k}_g_nb"]) <= 1e-5


def test_fully_masked_row_is_uniform():
    """src/attention.py:151-161: a fully-masked query row attends uniformly."""
    g = load_golden("attn_ops.npz")
    x, mask, nb, p = _attn_case(g, 2)
    _, cache = O.attention_fwd(x, mask, nb, p)
    w = cache["w"]  # [B,S,H,R,R]; row s=0 fully masked
    assert np.allclose(w[0, 0], 1.0 / w.shape[-1], atol=1e-7)


@pytest.mark.parametrize("fname", ["model_O.npz", "model_O_h4.npz", "model_mini.npz"])
def test_model_grads_match_reference(fname):
    g = load_golden(fname)
    nb, s, r, cm, cz, h, k, ncyc, fseed, pseed = (int(v) for v in g["cfg"])
    cfg = O.ModelConfig(n_blocks=nb, n_seq=s, n_res=r, c_m=cm, c_z=cz, heads=h, opm_dim=k)
    P = O.init_params(cfg, pseed)
    feats = O.make_features(cfg, fseed)
    assert np.array_equal(feats.msa_feat, g["msa_feat"])
    assert np.array_equal(feats.pair_feat, g["pair_feat"])
    loss, grads, (msa, pair) = O.serial_grads(cfg, P, feats, ncyc)
    assert abs(loss - float(g["loss"])) <= 1e-6 * max(1.0, abs(float(g["loss"])))
    assert rel_err(msa, g["msa"]) <= 1e-5
    assert rel_err(pair, g["pair"]) <= 1e-5
    gmax = max(np.abs(g[f"g::{n}"]).max() for n in grads)
    worst = max(rel_err(grads[n], g[f"g::{n}"], 1e-6 * gmax) for n in grads)
    assert worst <= 1e-4, worst


def test_optimizer_matches_reference():
    g = load_golden("optim.npz")
    names = [f"p{i}" for i in range(7)]
    params = {n: g[f"init::{n}"].copy() for n in names}
    opt = O.FusedOptimizer(params)
    for step in range(4):
        norm = opt.apply({n: g[f"grad{step}::{n}"] for n in names})
        assert abs(norm - float(g[f"norm{step}"])) <= 1e-12 * norm
        for n in names:
            assert np.array_equal(params[n], g[f"param{step}::{n}"]), (step, n)
            assert np.array_equal(opt.ema[n], g[f"ema{step}::{n}"]), (step, n)


def test_layout_matches_reference_rule():
    """src/fusion.py:50-58: 256-B aligned, padded slots in flatten order."""
    lay = O.build_layout([("a", (5,)), ("b", (7, 3)), ("c", (1,)), ("d", ())])
    assert [x[2] for x in lay] == [0, 256, 512, 768]
    assert all(x[4] % 256 == 0 and x[4] >= x[3] for x in lay)
