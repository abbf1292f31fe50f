"""DAP (src/harness.py:262-293, 355-389) on the sm_100a engine.

The ranks are processes sharing the one GPU of the test box over a gloo group
(``Comm`` stages device buffers through host memory there; NCCL runs the same
calls on device buffers).  Each rank computes its shard's forward and
backward with the CUDA kernels; the synced gradients, the loss and the
gathered outputs must match the unsharded engine on the same GPU
(tests/test_acceptance.py:184-198 of the reference: parallel transparency),
and the per-block collective counts must match the planner's mini table
(src/planner.py:46-50; tests/test_acceptance.py:168-181)."""

import os
import socket
import tempfile
from collections import Counter

import numpy as np
import pytest

from conftest import rel_err, slot_errs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CFGS = {
    "mini": dict(n_blocks=2, n_seq=16, n_res=32, c_m=64, c_z=32, heads=2, opm_dim=8),
    "k32": dict(n_blocks=1, n_seq=32, n_res=64, c_m=64, c_z=32, heads=2, opm_dim=32),
    # L = 128 / 96 reach the tcgen05 attention kernels in bf16
    "tc": dict(n_blocks=1, n_seq=96, n_res=128, c_m=64, c_z=64, heads=2, opm_dim=32),
}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_05477_b200 import _lib
    _lib.lib()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _build(cfg_kw, dtype_name):
    from paper_2207_05477_b200.fusion import FusionEngine
    from paper_2207_05477_b200.model import ModelConfig, flatten_params, init_params
    cfg = ModelConfig(**cfg_kw)
    P = init_params(cfg, 7)
    dt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
    st = FusionEngine([(n, P[n]) for n, _ in flatten_params(cfg)], shadow_dtype=dt)
    return cfg, st, dt


def _worker(rank, world, port, cfg_kw, dtype_name, n_cycles, recompute, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2207_05477_b200.dap import DapEngine, dap_step
    from paper_2207_05477_b200.engine import DeviceFeatures
    from paper_2207_05477_b200.model import make_features
    from paper_2207_05477_b200.parallel import GridConfig, build_dap_groups
    cfg, st, dt = _build(cfg_kw, dtype_name)
    grid = GridConfig(dap=world)
    dap, world_comm = build_dap_groups(grid)
    eng = DapEngine(cfg, st, dt, dap)
    feats = DeviceFeatures(make_features(cfg, 3), "cuda", cfg)
    loss, (msa, pair) = dap_step(eng, feats, world_comm, grid, n_cycles=n_cycles, recompute=recompute)
    fm, fp = eng.gather_outputs(msa, pair)
    torch.cuda.synchronize()
    if rank == 0:
        recs = [(r.module, r.primitive, r.phase) for r in dap.records]
        np.savez(out_path, loss=loss.cpu().numpy(), grads=st.regions["grads"].cpu().numpy(),
                 msa=fm.float().cpu().numpy(), pair=fp.float().cpu().numpy(),
                 recs=np.array(recs, dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def _run_dap(world, cfg_kw, dtype_name, n_cycles=1, recompute=False):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r.npz")
        mp.spawn(_worker, args=(world, _free_port(), cfg_kw, dtype_name, n_cycles, recompute, out),
                 nprocs=world, join=True)
        r = np.load(out, allow_pickle=True)
        return {k: r[k] for k in r.files}


def _run_serial(cfg_kw, dtype_name, n_cycles=1):
    from paper_2207_05477_b200.engine import BlockEngine, DeviceFeatures
    from paper_2207_05477_b200.model import make_features
    cfg, st, dt = _build(cfg_kw, dtype_name)
    eng = BlockEngine(cfg, st, dt)
    feats = DeviceFeatures(make_features(cfg, 3), "cuda", cfg)
    loss, (msa, pair) = eng.forward_backward(feats, n_cycles)
    torch.cuda.synchronize()
    return dict(loss=loss.cpu().numpy(), grads=st.regions["grads"].cpu().numpy(),
                msa=msa.float().cpu().numpy(), pair=pair.float().cpu().numpy(), store=st)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("world,cfg,dtype,ncyc", [
    (2, "mini", "f32", 1), (4, "mini", "f32", 1), (2, "mini", "f32", 2), (2, "k32", "f32", 1),
    (2, "tc", "bf16", 1)])
def test_dap_matches_unsharded(world, cfg, dtype, ncyc):
    kw = CFGS[cfg]
    base = _run_serial(kw, dtype, ncyc)
    res = _run_dap(world, kw, dtype, ncyc)
    tol = 1e-4 if dtype == "f32" else 3e-2
    S, R = kw["n_seq"], kw["n_res"]
    assert abs(float(res["loss"][0]) - float(base["loss"][0])) <= tol * abs(float(base["loss"][0]))
    assert rel_err(res["msa"].reshape(S * R, -1), base["msa"]) <= tol
    assert rel_err(res["pair"].reshape(R * R, -1), base["pair"]) <= tol
    # per parameter, floored (a DAP partial never reduced would show here)
    errs = slot_errs(base["store"], res["grads"], base["grads"], 1e-6 if dtype == "f32" else 1e-3)
    worst = max(errs, key=errs.get)
    assert errs[worst] <= (tol if dtype == "f32" else 5e-2), (worst, errs[worst])
    if dtype == "f32":  # and against the CPU oracle itself
        from oracle import evoformer_np as O
        ocfg = O.ModelConfig(**kw)
        oloss, ograds, (omsa, opair) = O.serial_grads(ocfg, O.init_params(ocfg, 7), O.make_features(ocfg, 3),
                                                     n_cycles=ncyc)
        assert abs(float(res["loss"][0]) - oloss) <= 1e-4 * abs(oloss)
        assert rel_err(res["pair"].reshape(opair.shape), opair) <= 1e-4
        errs = slot_errs(base["store"], res["grads"], ograds, 1e-6)
        worst = max(errs, key=errs.get)
        assert errs[worst] <= 1e-4, (worst, errs[worst])


@pytest.mark.timeout(600)
def test_dap_trace_matches_planner_mini_table():
    kw = CFGS["mini"]
    from paper_2207_05477_b200 import planner
    res = _run_dap(2, kw, "f32")
    measured = planner.trace_counts([tuple(r) for r in res["recs"]])
    assert measured == planner.expected_trace("dap", kw["n_blocks"], "mini")
    # everything after the loss is backward traffic: half of each block's all-to-alls
    phases = Counter(ph for m, pr, ph in map(tuple, res["recs"]) if pr == "alltoall")
    assert phases["fwd"] == phases["bwd"] == 4 * kw["n_blocks"]


@pytest.mark.timeout(600)
def test_dap_recompute_bitwise():
    kw = CFGS["mini"]
    a = _run_dap(2, kw, "f32")
    b = _run_dap(2, kw, "f32", recompute=True)
    assert np.array_equal(a["grads"], b["grads"]) and np.array_equal(a["loss"], b["loss"])
