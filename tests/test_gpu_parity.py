"""GPU parity: the sm_100a path against the CPU oracle and the reference goldens.

fp32 mode: every output and gradient within rtol 1e-4 (floored inf-norm,
SURVEY.md section 8c).  bf16 mode: outputs within 3e-2 and gradients within
5e-2 of the fp32 oracle (the reference's own bf16 acceptance bound is 3e-2,
tests/test_acceptance.py:304-318 of the reference).
"""

import numpy as np
import pytest

from conftest import load_golden, rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4
BF16_OUT_TOL = 3e-2
BF16_GRAD_TOL = 5e-2


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_05477_b200 import _lib
    _lib.lib()  # raises if the library is missing or the device is not sm_100


def _model_case(fname):
    from paper_2207_05477_b200.model import ModelConfig
    g = load_golden(fname)
    nb, s, r, cm, cz, h, k, ncyc, fseed, pseed = (int(v) for v in g["cfg"])
    cfg = ModelConfig(n_blocks=nb, n_seq=s, n_res=r, c_m=cm, c_z=cz, heads=h, opm_dim=k)
    return g, cfg, ncyc, fseed, pseed


def _run_engine(cfg, pseed, fseed, ncyc, dtype):
    from paper_2207_05477_b200.engine import BlockEngine, DeviceFeatures
    from paper_2207_05477_b200.fusion import FusionEngine
    from paper_2207_05477_b200.model import flatten_params, init_params, make_features
    P = init_params(cfg, pseed)
    st = FusionEngine([(n, P[n]) for n, _ in flatten_params(cfg)], shadow_dtype=dtype)
    eng = BlockEngine(cfg, st, dtype)
    feats = DeviceFeatures(make_features(cfg, fseed), "cuda", cfg)
    loss, (msa, pair) = eng.forward_backward(feats, ncyc)
    torch.cuda.synchronize()
    grads = {n: st.grad(n).cpu().numpy() for n, _ in flatten_params(cfg)}
    return float(loss.item()), msa.float().cpu().numpy(), pair.float().cpu().numpy(), grads


@pytest.mark.parametrize("fname", ["model_O.npz", "model_O_h4.npz", "model_mini.npz"])
def test_block_fp32_matches_reference(fname):
    g, cfg, ncyc, fseed, pseed = _model_case(fname)
    loss, msa, pair, grads = _run_engine(cfg, pseed, fseed, ncyc, torch.float32)
    S, R = cfg.n_seq, cfg.n_res
    assert rel_err(msa.reshape(g["msa"].shape), g["msa"]) <= FP32_TOL
    assert rel_err(pair.reshape(g["pair"].shape), g["pair"]) <= FP32_TOL
    assert abs(loss - float(g["loss"])) <= FP32_TOL * abs(float(g["loss"]))
    gmax = max(np.abs(g[f"g::{n}"]).max() for n in grads)
    errs = {n: rel_err(grads[n], g[f"g::{n}"], 1e-6 * gmax) for n in grads}
    worst = max(errs, key=errs.get)
    assert errs[worst] <= FP32_TOL, (worst, errs[worst])


@pytest.mark.parametrize("fname", ["model_O.npz", "model_O_h4.npz"])
def test_block_bf16_within_bound(fname):
    g, cfg, ncyc, fseed, pseed = _model_case(fname)
    loss, msa, pair, grads = _run_engine(cfg, pseed, fseed, ncyc, torch.bfloat16)
    assert rel_err(msa.reshape(g["msa"].shape), g["msa"]) <= BF16_OUT_TOL
    assert rel_err(pair.reshape(g["pair"].shape), g["pair"]) <= BF16_OUT_TOL
    gmax = max(np.abs(g[f"g::{n}"]).max() for n in grads)
    errs = {n: rel_err(grads[n], g[f"g::{n}"], 1e-3 * gmax) for n in grads}
    worst = max(errs, key=errs.get)
    assert errs[worst] <= BF16_GRAD_TOL, (worst, errs[worst])


@pytest.mark.parametrize("k", range(6))
def test_attention_op_matches_reference(k):
    from paper_2207_05477_b200.attention import (AttentionInput, AttentionParams,
                                                 gated_attention_fused)
    g = load_golden("attn_ops.npz")
    seed, b, s, r, h, c, fm, use_bias = (int(v) for v in g[f"c{k}_meta"])
    dev = "cuda"

    def T(a, grad=True):
        t = torch.tensor(a, device=dev)
        return t.requires_grad_(grad)

    x = T(g[f"c{k}_x"])
    nb = T(g[f"c{k}_nb"]) if use_bias else None
    ps = AttentionParams(*[T(g[f"c{k}_p_{f}"]) for f in ("wq", "wk", "wv", "wg", "bg", "wo", "bo")])
    out = gated_attention_fused(AttentionInput(x, T(g[f"c{k}_mask"], False), nb), ps)
    loss = (out * out).mean()
    loss.backward()
    assert rel_err(out.detach().cpu().numpy(), g[f"c{k}_out"]) <= 1e-5
    assert rel_err(x.grad.cpu().numpy(), g[f"c{k}_g_x"]) <= FP32_TOL
    if use_bias:
        assert rel_err(nb.grad.cpu().numpy(), g[f"c{k}_g_nb"]) <= FP32_TOL
    for f, t in zip(("wq", "wk", "wv", "wg", "bg", "wo", "bo"), ps.all()):
        assert rel_err(t.grad.cpu().numpy(), g[f"c{k}_g_{f}"], 1e-8) <= FP32_TOL, f


def test_optimizer_bitwise_matches_reference():
    from paper_2207_05477_b200.fusion import FusionEngine
    g = load_golden("optim.npz")
    names = [f"p{i}" for i in range(7)]
    eng = FusionEngine([(n, g[f"init::{n}"]) for n in names], shadow_dtype=torch.bfloat16)
    for step in range(4):
        norm = eng.apply({n: g[f"grad{step}::{n}"] for n in names})
        assert abs(norm - float(g[f"norm{step}"])) <= 1e-12 * norm
        for n in names:
            assert np.array_equal(eng.param(n).cpu().numpy(), g[f"param{step}::{n}"]), (step, n)
            assert np.array_equal(eng.view("ema", n).cpu().numpy(), g[f"ema{step}::{n}"]), (step, n)
        sh = eng.view("shadow", names[0]).float().cpu().numpy()
        assert np.allclose(sh, eng.param(names[0]).cpu().numpy(), rtol=1e-2, atol=1e-6)


def test_fully_masked_rows_uniform_on_gpu():
    """A fully-masked query row must attend uniformly (reference semantics,
    src/attention.py:151-161) -- exercised through the attention golden with
    a fully-masked sequence (case 2) and directly here."""
    from paper_2207_05477_b200 import ops
    B, L, H, D = 2, 16, 2, 16
    qkvg = torch.randn(B * L, 4 * H * D, device="cuda")
    mask = torch.ones(B, L, device="cuda")
    mask[1] = 0.0
    bg = torch.zeros(H * D, device="cuda")
    ctx, gate, gated, lse = ops.attn_fwd(qkvg, mask, L, 1, None, bg, B, L, H, D, L, 1)
    v = qkvg[L:, 2 * H * D:3 * H * D]
    expect = v.mean(dim=0, keepdim=True).expand(L, -1)
    assert torch.allclose(ctx[L:], expect, atol=1e-5)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_block_with_trimul_matches_oracle(dtype):
    """TriangleMultiplication extension (AF2 Alg 11/12) against the oracle
    restatement -- parity UNPINNED (no reference code), so this checks the
    GPU path against the restatement, whose backward is FD-checked on CPU.

    Run at the oracle shape O: at smaller channel counts the pair-bias
    weight gradients (sums of softmax-gradient rows, which cancel) drift
    past the bf16 bound in the reference itself -- its own bf16-vs-fp32
    deviation at S=16, R=32, c_m=c_z=32 is 5.04e-2 on tri_end.w_bias, at O
    2.3e-2 (row_attn.w_bias), measured with the reference's act_dtype=BF16."""
    from oracle import evoformer_np as O
    from paper_2207_05477_b200.model import ModelConfig
    kw = dict(n_blocks=1, n_seq=32, n_res=64, c_m=64, c_z=32, heads=2, opm_dim=32, trimul=True)
    cfg = ModelConfig(**kw)
    ocfg = O.ModelConfig(**kw)
    oloss, ograds, (omsa, opair) = O.serial_grads(ocfg, O.init_params(ocfg, 7), O.make_features(ocfg, 3))
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    loss, msa, pair, grads = _run_engine(cfg, 7, 3, 1, dt)
    tol_o, tol_g, floor = (FP32_TOL, FP32_TOL, 1e-6) if dtype == "f32" else (BF16_OUT_TOL, BF16_GRAD_TOL, 1e-3)
    assert rel_err(pair.reshape(opair.shape), opair) <= tol_o
    assert rel_err(msa.reshape(omsa.shape), omsa) <= tol_o
    gmax = max(np.abs(v).max() for v in ograds.values())
    errs = {n: rel_err(grads[n], ograds[n], floor * gmax) for n in ograds}
    worst = max(errs, key=errs.get)
    assert errs[worst] <= tol_g, (worst, errs[worst])
    assert any("tri_mul" in n and np.abs(grads[n]).max() > 0 for n in grads)


def test_bench_shape_step_gradients_finite():
    """Two Evoformer blocks at the bench shape (N_seq=128, N_res=256, bf16,
    padded residues): one fwd+bwd gives a finite loss and finite gradients in
    every parameter slot (the small-shape parity tests cannot reach the
    many-batches-per-CTA attention paths this exercises)."""
    import torch
    from paper_2207_05477_b200.model import ModelConfig
    from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer
    cfg = ModelConfig(n_blocks=2, n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32)
    tr = Trainer.create(cfg, ExecutionPlan(act_dtype="bf16", fixed_recycles=1))
    loss, _ = tr.engine.forward_backward(tr.feats, 1)
    torch.cuda.synchronize()
    assert np.isfinite(float(loss))
    bad = [n for n in tr.store.names if not bool(torch.isfinite(tr.store.grad(n)).all())]
    assert not bad, bad[:5]


@pytest.mark.parametrize("dtype,streams,nb,s,r", [
    ("f32", True, 3, 16, 32), ("bf16", True, 3, 16, 32), ("bf16", False, 3, 16, 32),
    ("bf16", True, 2, 128, 256)])
def test_recompute_grads_bitwise_equal_direct(dtype, streams, nb, s, r):
    """src/trainer.py:108-179: storing only block inputs and recomputing each
    block's forward during the backward gives bitwise the loss and gradients
    of the stored-activation pass (two recycles: the untaped pass feeds in)."""
    from paper_2207_05477_b200.model import ModelConfig
    from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer
    if r == 256:
        cfg = ModelConfig(n_blocks=nb, n_seq=s, n_res=r, c_m=256, c_z=128, heads=8, opm_dim=32)
    else:
        cfg = ModelConfig(n_blocks=nb, n_seq=s, n_res=r, c_m=64, c_z=32, heads=2, opm_dim=8)
    out = []
    for rc in ((), ("evoformer",)):
        tr = Trainer.create(cfg, ExecutionPlan(act_dtype=dtype, recompute=rc, fixed_recycles=2))
        tr.engine.branch_streams = streams
        loss, (msa, pair) = tr.engine.forward_backward(tr.feats, 2, recompute=tr.plan.recompute_on)
        torch.cuda.synchronize()
        out.append((loss.cpu(), msa.cpu(), pair.cpu(),
                    {n: tr.store.grad(n).cpu() for n in tr.store.names}))
    (l0, m0, p0, g0), (l1, m1, p1, g1) = out
    assert torch.equal(l0, l1) and torch.equal(m0, m1) and torch.equal(p0, p1)
    diff = [n for n in g0 if not torch.equal(g0[n], g1[n])]
    assert not diff, diff[:5]
    assert any(bool(g.abs().max() > 0) for g in g0.values())


def test_train_loop_metrics_jsonl_and_bench_protocol(tmp_path):
    """src/trainer.py:192-303: per-step metrics (fused optimizer = 1/2/1/1
    launches per phase, src/planner.py launches_per_step), metrics.jsonl, and
    the bench protocol's discarded prefix not leaking into the averages."""
    import json
    from paper_2207_05477_b200.model import ModelConfig
    from paper_2207_05477_b200.trainer import COUNTER_KEYS, ExecutionPlan, Trainer
    cfg = ModelConfig(n_blocks=2, n_seq=16, n_res=32, c_m=64, c_z=32, heads=2, opm_dim=8)
    tr = Trainer.create(cfg, ExecutionPlan(act_dtype="f32", seed=32))
    path = tmp_path / "metrics.jsonl"
    losses = tr.train_loop(3, str(path))
    lines = [json.loads(x) for x in path.read_text().splitlines()]
    assert [m["step"] for m in lines] == [0, 1, 2]
    assert [m["loss"] for m in lines] == losses and all(np.isfinite(losses))
    for m in lines:
        assert m["launches"] == {"grad_sync": 1, "grad_clip": 2, "opt_update": 1, "ema": 1}
        assert set(COUNTER_KEYS) <= set(m)
        assert m["op_count"] > 0 and m["ledger_peak_bytes"] > 0
        assert m["blocks_executed"] == cfg.n_blocks * m["n_recycles"]
    tr2 = Trainer.create(cfg, ExecutionPlan(act_dtype="f32", seed=32))
    rep = tr2.bench_protocol(total=4, discard=1, _spike=(0, "loss", 1e6))
    assert rep["averaged_steps"] == 3
    kept = tr2.history[1:]
    assert abs(rep["counters"]["loss"] - np.mean([m["loss"] for m in kept])) <= 1e-6 * abs(rep["counters"]["loss"])
    assert rep["counters"]["launch_total"] == 5.0
