"""TriangleMultiplication restatement (AF2 Supplementary Alg. 11/12).

The reference has no TriangleMultiplication code (planner inventory only,
src/planner.py:37-45), so this oracle's parity is UNPINNED.  What can be
checked without a reference: the hand-written backward against central finite
differences (the reference's own gradient-check methodology,
src/autodiff.py:125-161), and the algebraic definition of the two
contractions against an einsum restatement.
"""

import numpy as np
import pytest

from oracle import evoformer_np as O


def _setup(outgoing, seed=0, R=6, cz=8):
    cfg = O.ModelConfig(n_blocks=1, n_seq=4, n_res=R, c_m=8, c_z=cz, heads=2, opm_dim=2, trimul=True)
    P = O.init_params(cfg, 11)
    rng = np.random.default_rng(seed)
    prefix = "block0.tri_mul_out" if outgoing else "block0.tri_mul_in"
    # non-trivial biases / LN affine so every term is exercised
    for name, shape, _ in O.param_specs(cfg):
        if name.startswith(prefix):
            P[name] = (P[name] + rng.normal(0, 0.1, shape)).astype(np.float32)
    pair = rng.normal(0, 1, (1, R, R, cz)).astype(np.float32)
    mask = np.ones((1, R, R), np.float32)
    mask[:, -1, :] = 0.0
    mask[:, :, -1] = 0.0
    return cfg, P, prefix, pair, mask


@pytest.mark.parametrize("outgoing", [True, False])
def test_trimul_contraction_definition(outgoing):
    cfg, P, prefix, pair, mask = _setup(outgoing)
    out, cache = O.trimul_fwd(pair, mask, P, prefix, outgoing)
    ac, bc = cache[7], cache[8]  # channel-major a, b
    a = ac.transpose(1, 2, 0)
    b = bc.transpose(1, 2, 0)
    o = np.einsum("ikc,jkc->ijc", a, b) if outgoing else np.einsum("kic,kjc->ijc", a, b)
    ol, _ = O.ln_fwd(o[None], P[f"{prefix}.ln_out_g"], P[f"{prefix}.ln_out_b"])
    zl, _ = O.ln_fwd(pair, P[f"{prefix}.ln_in_g"], P[f"{prefix}.ln_in_b"])
    g = O.sigmoid(zl @ P[f"{prefix}.w_g"] + P[f"{prefix}.b_g"])
    ref = pair + g * (ol @ P[f"{prefix}.w_o"] + P[f"{prefix}.b_o"])
    assert np.allclose(out, ref, atol=1e-5)


@pytest.mark.parametrize("outgoing", [True, False])
def test_trimul_backward_finite_differences(outgoing):
    cfg, P, prefix, pair, mask = _setup(outgoing, seed=1)
    rng = np.random.default_rng(5)
    wout = rng.normal(0, 1, pair.shape).astype(np.float32)

    def loss(pr, PP):
        out, _ = O.trimul_fwd(pr, mask, PP, prefix, outgoing)
        return float(np.sum(out.astype(np.float64) * wout))

    out, cache = O.trimul_fwd(pair, mask, P, prefix, outgoing)
    grads = {}
    dpair = O.trimul_bwd(wout, cache, P, prefix, grads)
    h = 1e-2
    checks = [("pair", None)] + [(n, None) for n in grads]
    for name, _ in checks:
        base = pair if name == "pair" else P[name]
        ana = dpair if name == "pair" else grads[name]
        flat = base.reshape(-1)
        idx = rng.choice(flat.size, size=min(6, flat.size), replace=False)
        for k in idx:
            orig = flat[k]
            flat[k] = orig + h
            lp = loss(pair, P)
            flat[k] = orig - h
            lm = loss(pair, P)
            flat[k] = orig
            fd = (lp - lm) / (2 * h)
            a = float(ana.reshape(-1)[k])
            assert abs(a - fd) <= 2e-2 * max(1.0, abs(fd)), (name, k, a, fd)
