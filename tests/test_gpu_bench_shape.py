"""Parity at the benchmarked configuration (shape I).

The bench times the initial-training shape (N_seq=128, N_res=256, c_m=256,
c_z=128, 8 heads, opm 32, padded residues) in bf16 with the tcgen05
attention kernels, the tcgen05 GEMMs, the fused OPM kernels and the two
branch streams.  The small-shape golden tests cannot reach those kernel paths
(L <= 64 takes the SIMT attention kernels), so here one Evoformer block at
shape I is compared with the CPU oracle (oracle/evoformer_np.py, itself
pinned to the reference goldens) on the same init_params / make_features:

* bf16 engine vs the fp32 oracle: outputs <= 3e-2, every gradient <= 5e-2
  (per tensor, floored inf-norm with floor 1e-3 * G, G = max |grad| over
  all tensors; the reference's own
  bf16 acceptance bound is 3e-2, tests/test_acceptance.py:304-318);
* fp32 engine: outputs and loss <= 1e-4 of the fp32 oracle; every gradient
  within 1e-4 of the oracle evaluated in float64 (``serial_grads_f64``), or,
  where the fp32 oracle itself is further than that from the float64 answer
  (long reductions: the 65,536-term w_bias / transition-W1 gradients sit at
  1-3e-4, measured), no further than 1.5x the fp32 oracle's own deviation --
  i.e. the GPU is at least as accurate as the reference's fp32 arithmetic.

Also: CUDA-graph replayed training steps equal eager ones bitwise (Adam's step
counter lives on the device, src/fusion.py:189-211).
"""

import os

import numpy as np
import pytest

from conftest import grad_err, rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SHAPE_I = dict(n_blocks=1, n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32)
PSEED, FSEED = 7, 3


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_05477_b200 import _lib
    _lib.lib()


@pytest.fixture(scope="module")
def oracle_I64():
    """The same block in float64 (~1 min on the host)."""
    from oracle import evoformer_np as O
    ocfg = O.ModelConfig(**SHAPE_I)
    loss, grads, (msa, pair) = O.serial_grads_f64(ocfg, O.init_params(ocfg, PSEED), O.make_features(ocfg, FSEED))
    return float(loss), grads, msa, pair


@pytest.fixture(scope="module")
def oracle_I():
    """One oracle block fwd+bwd at shape I (fp32 numpy; ~10-20 s on the host)."""
    from oracle import evoformer_np as O
    ocfg = O.ModelConfig(**SHAPE_I)
    loss, grads, (msa, pair) = O.serial_grads(ocfg, O.init_params(ocfg, PSEED), O.make_features(ocfg, FSEED))
    return float(loss), grads, msa, pair


def _engine_I(dtype, streams=True):
    from paper_2207_05477_b200.engine import BlockEngine, DeviceFeatures
    from paper_2207_05477_b200.fusion import FusionEngine
    from paper_2207_05477_b200.model import ModelConfig, flatten_params, init_params, make_features
    cfg = ModelConfig(**SHAPE_I)
    P = init_params(cfg, PSEED)
    st = FusionEngine([(n, P[n]) for n, _ in flatten_params(cfg)], shadow_dtype=dtype)
    eng = BlockEngine(cfg, st, dtype)
    eng.branch_streams = streams
    feats = DeviceFeatures(make_features(cfg, FSEED), "cuda", cfg)
    loss, (msa, pair) = eng.forward_backward(feats, 1)
    torch.cuda.synchronize()
    grads = {n: st.grad(n).cpu().numpy() for n in st.names}
    return float(loss.item()), msa.float().cpu().numpy(), pair.float().cpu().numpy(), grads


def _check(res, ref, tol_out, tol_grad, floor):
    loss, msa, pair, grads = res
    oloss, ograds, omsa, opair = ref
    e_msa = rel_err(msa.reshape(omsa.shape), omsa)
    e_pair = rel_err(pair.reshape(opair.shape), opair)
    assert e_msa <= tol_out, ("msa", e_msa)
    assert e_pair <= tol_out, ("pair", e_pair)
    assert abs(loss - oloss) <= tol_out * abs(oloss), (loss, oloss)
    gmax = max(float(np.abs(g).max()) for g in ograds.values())   # G of SURVEY section 8c
    errs = {n: grad_err(grads[n].reshape(g.shape), g, n, floor, gmax) for n, g in ograds.items()}
    worst = max(errs, key=errs.get)
    assert errs[worst] <= tol_grad, (worst, errs[worst], sorted(errs.values())[-5:])
    # every slot the oracle gives a gradient got one (recycling parameters
    # have none with one cycle; bias_ln_b is analytically zero)
    dead = [n for n, g in ograds.items() if np.abs(g).max() > 1e-6 * gmax and not np.abs(grads[n]).max() > 0]
    assert not dead, dead


def test_bench_shape_bf16_matches_oracle(oracle_I):
    _check(_engine_I(torch.bfloat16), oracle_I, 3e-2, 5e-2, 1e-3)


def test_bench_shape_bf16_single_stream_matches_oracle(oracle_I):
    _check(_engine_I(torch.bfloat16, streams=False), oracle_I, 3e-2, 5e-2, 1e-3)


def test_bench_shape_fp32_matches_oracle(oracle_I, oracle_I64):
    loss, msa, pair, grads = _engine_I(torch.float32)
    oloss, ograds, omsa, opair = oracle_I
    _, g64, _, _ = oracle_I64
    assert rel_err(msa.reshape(omsa.shape), omsa) <= 1e-4
    assert rel_err(pair.reshape(opair.shape), opair) <= 1e-4
    assert abs(loss - oloss) <= 1e-4 * abs(oloss)
    G = max(float(np.abs(g).max()) for g in g64.values())
    bad = {}
    for n, g in g64.items():
        e_gpu = grad_err(grads[n].reshape(g.shape), g, n, 1e-6, G)
        e_ref = grad_err(ograds[n], g, n, 1e-6, G)      # the fp32 oracle's own rounding
        if e_gpu > max(1e-4, 1.5 * e_ref):
            bad[n] = (e_gpu, e_ref)
    assert not bad, bad


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_graph_replay_equals_eager_bitwise(dtype):
    """N CUDA-graph replays of the captured training step == N eager steps,
    bitwise in params, Adam moments, EMA and the bf16 shadow (the bias
    corrections 1 - beta^t must advance on replay)."""
    from paper_2207_05477_b200.model import ModelConfig
    from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer
    cfg = ModelConfig(n_blocks=2, n_seq=16, n_res=64, c_m=64, c_z=32, heads=2, opm_dim=8)
    steps = 5
    eager = Trainer.create(cfg, ExecutionPlan(act_dtype=dtype, fixed_recycles=1))
    for _ in range(steps):
        eager.device_step(1, h2d=False)
    graph = Trainer.create(cfg, ExecutionPlan(act_dtype=dtype, fixed_recycles=1))
    graph.capture(n_cycles=1, warmup=1)
    for _ in range(steps - 1):
        graph.replay()
    torch.cuda.synchronize()
    assert eager.store.step_count == graph.store.step_count == steps
    assert graph.store.device_step_count() == steps
    for r in ("params", "adam_m", "adam_v", "ema"):
        assert torch.equal(eager.store.regions[r], graph.store.regions[r]), r
    if eager.store.shadow is not None:
        assert torch.equal(eager.store.shadow, graph.store.shadow)
    # and one more eager step after replays continues the same trajectory
    eager.device_step(1, h2d=False)
    graph.device_step(1, h2d=False)
    torch.cuda.synchronize()
    assert torch.equal(eager.store.regions["params"], graph.store.regions["params"])
