"""Parity beyond the bench shape (SURVEY.md section 8 configs[4], A4, A5 and (f)1).

* Fine-tune shape F (N_seq=512, N_res=384): one Evoformer block fwd+bwd in
  bf16 against the fp32 CPU oracle.  Rows longer than 256 keys take the
  key-blocked tcgen05 forward and the key-window backward (row attention
  L=384, column attention L=512), which the bench shape never reaches.
  Bound: outputs <= 3e-2, every gradient <= 5e-2 (per tensor, floored
  inf-norm, floor 1e-3 G) -- the bench-shape bound of test_gpu_bench_shape.py.
* Inference stress shape X (N_res=1024): triangle attention (starting node,
  4 heads of 32, padded residues) through ``subbatch_apply`` with chunk 32
  (src/attention.py:236-267) on a 64-row subset, bf16 against the oracle's
  ``gated_attention_fused`` forward (src/attention.py:121-174) on the same rows.
* ``gated_attention_reference`` (A4): the unfused fp32 baseline with
  materialised logits, forward and gradients against the oracle.
"""

import numpy as np
import pytest

from conftest import grad_err, rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SHAPE_F = dict(n_blocks=1, n_seq=512, n_res=384, c_m=256, c_z=128, heads=8, opm_dim=32)
PSEED, FSEED = 11, 5


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_05477_b200 import _lib
    _lib.lib()


def test_fine_tune_shape_block_bf16_matches_oracle():
    from oracle import evoformer_np as O
    from paper_2207_05477_b200.engine import BlockEngine, DeviceFeatures
    from paper_2207_05477_b200.fusion import FusionEngine
    from paper_2207_05477_b200.model import ModelConfig, flatten_params, init_params, make_features

    cfg = ModelConfig(**SHAPE_F)
    P = init_params(cfg, PSEED)
    st = FusionEngine([(n, P[n]) for n, _ in flatten_params(cfg)], shadow_dtype=torch.bfloat16)
    eng = BlockEngine(cfg, st, torch.bfloat16)
    feats = DeviceFeatures(make_features(cfg, FSEED), "cuda", cfg)
    loss, (msa, pair) = eng.forward_backward(feats, 1)
    torch.cuda.synchronize()
    grads = {n: st.grad(n).cpu().numpy() for n in st.names}
    msa, pair, loss = msa.float().cpu().numpy(), pair.float().cpu().numpy(), float(loss.item())

    ocfg = O.ModelConfig(**SHAPE_F)
    oloss, ograds, (omsa, opair) = O.serial_grads(ocfg, O.init_params(ocfg, PSEED), O.make_features(ocfg, FSEED))
    assert rel_err(msa.reshape(omsa.shape), omsa) <= 3e-2
    assert rel_err(pair.reshape(opair.shape), opair) <= 3e-2
    assert abs(loss - oloss) <= 3e-2 * abs(oloss)
    gmax = max(float(np.abs(g).max()) for g in ograds.values())
    errs = {n: grad_err(grads[n].reshape(g.shape), g, n, 1e-3, gmax) for n, g in ograds.items()}
    worst = max(errs, key=errs.get)
    assert errs[worst] <= 5e-2, (worst, errs[worst])


def _attn_params(rng, C, H, D, dev=True):
    shapes = ((C, H, D),) * 4 + ((H, D), (H, D, C), (C,))
    scales = (C ** -0.5,) * 4 + (0.5, (H * D) ** -0.5, 0.1)
    arrs = [(s * rng.standard_normal(sh)).astype(np.float32) for sh, s in zip(shapes, scales)]
    return arrs


def test_inference_shape_tri_attention_subbatch_matches_oracle():
    """X: N_res = 1024, starting-node triangle attention of 64 rows i (all
    1024 keys j per row), chunked 32 rows at a time."""
    from oracle import evoformer_np as O
    from paper_2207_05477_b200.attention import (AttentionInput, AttentionParams, gated_attention_fused,
                                                 subbatch_apply)
    rng = np.random.default_rng(1024)
    R, C, H, D, NI = 1024, 128, 4, 32, 64
    x = rng.standard_normal((1, NI, R, C)).astype(np.float32)
    mask = np.ones((1, NI, R), np.float32)
    mask[:, :, 1000:] = 0.0          # padded residues
    mask[:, 3, :] = 0.0              # one fully-masked row (uniform attention)
    nb = (0.5 * rng.standard_normal((H, R, R))).astype(np.float32)
    nb = O.bf16_round(nb)            # the device operator stores the bias in bf16
    pa = _attn_params(rng, C, H, D)
    ref, _ = O.attention_fwd(x, mask, nb, dict(zip(("wq", "wk", "wv", "wg", "bg", "wo", "bo"), pa)))

    dev = lambda a: torch.from_numpy(a).cuda()
    p = AttentionParams(*[dev(a) for a in pa])
    nb_t = dev(nb)
    f = lambda xc, mc: gated_attention_fused(AttentionInput(xc, mc, nb_t), p, act_dtype=torch.bfloat16)
    with torch.no_grad():
        out = subbatch_apply(f, dev(x), 1, 32, companions=(dev(mask),))
    torch.cuda.synchronize()
    assert out.shape == (1, NI, R, C)
    assert rel_err(out.cpu().numpy(), ref) <= 3e-2


def test_gated_attention_reference_unfused_fwd_bwd():
    """``gated_attention_reference`` (src/attention.py:78-115): the unfused
    fp32 composition with materialised [B*S, H, R, R] logits on the library's
    GEMM / softmax / gate kernels.  Forward and every gradient against the
    oracle (the reference's own parity bound for the pair: forward 1e-5,
    gradients 1e-4, tests/test_acceptance.py:46-71), and against the fused
    operator in fp32 and bf16."""
    from oracle import evoformer_np as O
    from paper_2207_05477_b200.attention import (AttentionInput, AttentionParams, gated_attention_fused,
                                                 gated_attention_reference)
    rng = np.random.default_rng(7)
    S, R, C, H, D = 6, 80, 64, 4, 16
    x = rng.standard_normal((1, S, R, C)).astype(np.float32)
    mask = np.ones((1, S, R), np.float32)
    mask[:, :, 70:] = 0.0
    mask[:, 2, :] = 0.0                      # a fully-masked row
    nb = (0.5 * rng.standard_normal((H, R, R))).astype(np.float32)
    names = ("wq", "wk", "wv", "wg", "bg", "wo", "bo")
    pa = _attn_params(rng, C, H, D)
    ref, cache = O.attention_fwd(x, mask, nb, dict(zip(names, pa)))
    gout = rng.standard_normal(ref.shape).astype(np.float32)
    odx, odp, odnb = O.attention_bwd(gout, cache)
    ograds = dict(odp, x=odx, nb=odnb)

    dev = lambda a, g=True: torch.from_numpy(a).cuda().requires_grad_(g)
    xt, nbt = dev(x), dev(nb)
    pt = AttentionParams(*[dev(a) for a in pa])
    out = gated_attention_reference(AttentionInput(xt, dev(mask, False), nbt), pt)
    out.backward(torch.from_numpy(gout).cuda())
    torch.cuda.synchronize()
    assert rel_err(out.detach().cpu().numpy(), ref) <= 1e-5
    got = dict(zip(("x", "nb") + names, [t.grad.cpu().numpy() for t in (xt, nbt, *pt.all())]))
    for name in ("x", "nb") + names:
        want = ograds[name]
        assert rel_err(got[name].reshape(want.shape), want) <= 1e-4, name
    with torch.no_grad():
        inp = AttentionInput(xt.detach(), dev(mask, False), nbt.detach())
        pd = AttentionParams(*[t.detach() for t in pt.all()])
        fused32 = gated_attention_fused(inp, pd)
        fused16 = gated_attention_fused(inp, pd, act_dtype=torch.bfloat16)
    assert rel_err(fused32.cpu().numpy(), out.detach().cpu().numpy()) <= 1e-5
    assert rel_err(fused16.float().cpu().numpy(), out.detach().cpu().numpy()) <= 3e-2
