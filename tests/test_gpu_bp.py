"""Branch Parallelism and DP (src/harness.py:392-616) on the sm_100a engine.

As in test_gpu_dap.py, the ranks are processes sharing the test box's one
GPU over a gloo group (device buffers staged through host memory; NCCL takes
them in place).  The synced gradients and the loss of a bp2 and a dp2 x bp2
step must match the unsharded engine (tests/test_acceptance.py:184-198 of the
reference), and each block must record the reference's 3 broadcasts + 1
all-reduce (tests/test_acceptance.py:156-166)."""

import os
import tempfile

import numpy as np
import pytest

from conftest import slot_errs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CFG = dict(n_blocks=2, n_seq=16, n_res=32, c_m=64, c_z=32, heads=2, opm_dim=8)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_05477_b200 import _lib
    _lib.lib()


def _engine(dtype_name):
    from paper_2207_05477_b200.engine import BlockEngine, DeviceFeatures
    from paper_2207_05477_b200.fusion import FusionEngine
    from paper_2207_05477_b200.model import ModelConfig, flatten_params, init_params, make_features
    cfg = ModelConfig(**CFG)
    P = init_params(cfg, 7)
    dt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
    st = FusionEngine([(n, P[n]) for n, _ in flatten_params(cfg)], shadow_dtype=dt)
    eng = BlockEngine(cfg, st, dt)
    return cfg, st, eng, DeviceFeatures(make_features(cfg, 3), "cuda", cfg)


def _worker(rank, world, port, dtype_name, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2207_05477_b200.parallel import GridConfig, bp_step, build_groups
    cfg, st, eng, feats = _engine(dtype_name)
    grid = GridConfig.for_world(world)
    bp, world_comm = build_groups(grid)
    loss = bp_step(eng, feats, bp, world_comm, grid, cfg.n_blocks)
    torch.cuda.synchronize()
    if rank == 0:
        recs = [(r.module, r.primitive) for r in bp.records]
        np.savez(out_path, loss=loss.cpu().numpy(), grads=st.regions["grads"].cpu().numpy(),
                 recs=np.array(recs, dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def _run(world, dtype_name):
    import torch.multiprocessing as mp
    from test_gpu_dap import _free_port
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r.npz")
        mp.spawn(_worker, args=(world, _free_port(), dtype_name, out), nprocs=world, join=True)
        r = np.load(out, allow_pickle=True)
        return {k: r[k] for k in r.files}


@pytest.mark.timeout(900)
@pytest.mark.parametrize("world,dtype", [(2, "f32"), (4, "f32"), (2, "bf16")])
def test_bp_matches_unsharded(world, dtype):
    _, st, eng, feats = _engine(dtype)
    loss, _ = eng.forward_backward(feats, 1)
    torch.cuda.synchronize()
    base_loss, base_g = float(loss.item()), st.regions["grads"].cpu().numpy()
    res = _run(world, dtype)
    tol = 1e-4 if dtype == "f32" else 3e-2
    assert abs(float(res["loss"][0]) - base_loss) <= tol * abs(base_loss)
    # per parameter, floored: a BP-pair gradient summed on both ranks or a
    # branch slot never synced would show here
    errs = slot_errs(st, res["grads"], base_g, 1e-6 if dtype == "f32" else 1e-3)
    worst = max(errs, key=errs.get)
    assert errs[worst] <= (tol if dtype == "f32" else 5e-2), (worst, errs[worst])
    if dtype == "f32":  # and against the CPU oracle itself, not only the unsharded engine
        from oracle import evoformer_np as O
        ocfg = O.ModelConfig(**CFG)
        oloss, ograds, _ = O.serial_grads(ocfg, O.init_params(ocfg, 7), O.make_features(ocfg, 3))
        assert abs(float(res["loss"][0]) - oloss) <= 1e-4 * abs(oloss)
        errs = slot_errs(st, res["grads"], ograds, 1e-6)
        worst = max(errs, key=errs.get)
        assert errs[worst] <= 1e-4, (worst, errs[worst])
    block = [r for r in map(tuple, res["recs"]) if r[0] in ("opm", "msa_stack", "pair_stack")]
    assert len(block) == 4 * CFG["n_blocks"]
    assert sum(1 for r in block if r[1] == "broadcast") == 3 * CFG["n_blocks"]


@pytest.mark.timeout(900)
def test_bench_multirank_bp_comm_trace(tmp_path):
    """``bench.py --gpus 2`` spawns its own ranks (torchrun-equivalent, here
    two ranks sharing the box's one GPU over gloo) and runs the BP step through
    Trainer.attach_parallel; each rank's CommRecord trace is written with the
    reference's CSV columns (src/harness.py:91-101) and the JSON line carries
    the per-step record count: 3 broadcasts + 1 all-reduce per block, the
    closing d(msa) broadcast and the grad all-reduce."""
    import csv
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pattern = str(tmp_path / "comm_r{rank}.csv")
    env = dict(os.environ, EVO_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2",
                          "--warmup", "1", "--blocks", "2", "--no-cpu-baseline", "--comm-csv", pattern],
                         cwd=root, env=env, capture_output=True, text=True, timeout=840)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "dp1xbp2"
    comm = line["comm"]
    per_block, closing = 4, 2          # opm, msa', pair' broadcasts + d(pair) all-reduce; msa_grad + grad_sync
    assert comm["records_per_step"] == 2 * per_block + closing, comm
    for r in range(2):
        rows = list(csv.reader(open(pattern.format(rank=r))))
        assert rows[0] == ["step", "phase", "group_axis", "group_id", "seq", "primitive", "bytes", "module"]
        body = rows[1:]
        assert len(body) == comm["records"]
        assert {b[1] for b in body} == {"fwd", "bwd", "grad-sync"}
        fwd = [b for b in body if b[0] == "0" and b[1] == "fwd"]
        assert [b[7] for b in fwd] == ["opm", "msa_stack", "pair_stack"] * 2
