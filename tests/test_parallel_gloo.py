"""Multi-process (gloo, CPU) tests of the branch-parallel / data-parallel
schedule in paper_2207_05477_b200/parallel.py.

The schedule is engine-agnostic; here each rank drives it with an adapter
around the CPU oracle (test infrastructure), so the collectives, the branch
split, the d(pair_in) all-reduce algebra (src/harness.py:500-515) and the
fused gradient all-reduce are checked against the serial oracle exactly as
the reference checks its thread grid (tests/test_harness.py:168-205 of the
reference): gradients / outputs / loss within 1e-5, and the per-block trace
of 3 broadcasts + 1 all-reduce.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import evoformer_np as O


def mini_cfg(n_blocks=2):
    return O.ModelConfig(n_blocks=n_blocks, n_seq=8, n_res=16, c_m=32, c_z=16, heads=4, opm_dim=4)


class OracleEngine:
    """The BlockEngine protocol of parallel.py, on the numpy oracle."""

    def __init__(self, cfg, P, feats):
        self.cfg, self.P, self.f = cfg, P, feats
        self.masks = O.make_masks(feats)
        self.specs = O.param_specs(cfg)
        self.grads = {}
        self.flat = None

    @staticmethod
    def T(a):
        return torch.from_numpy(np.ascontiguousarray(a, np.float32))

    def zero_grads(self):
        self.grads = {}

    def grad_region(self):
        parts = [np.asarray(self.grads.get(n, np.zeros(s, np.float32)), np.float32).ravel()
                 for n, s, _ in self.specs]
        self.flat = torch.from_numpy(np.concatenate(parts))
        return self.flat

    def empty_like(self, t):
        return torch.empty_like(t)

    def zeros_like(self, t):
        return torch.zeros_like(t)

    def add(self, a, b):
        return a + b

    def forward_only(self, feats, prev=None):
        prev_np = None if prev is None else (prev[0].numpy(), prev[1].numpy())
        m, p = O.model_forward(self.cfg, self.P, self.f, prev_np)
        return self.T(m), self.T(p)

    def embed_fwd(self, feats, prev=None):
        prev_np = None if prev is None else (prev[0].numpy(), prev[1].numpy())
        m, p, rc = O.embed_fwd(self.f, self.P, prev_np)
        return self.T(m), self.T(p), rc

    def opm_fwd(self, msa_in, prefix, feats, pair_res=None):
        out, c = O.opm_fwd(msa_in.numpy(), self.masks.msa, self.P, prefix, self.cfg.opm_dim)
        return self.T(out), c

    def msa_branch_fwd(self, i, msa_in, pair_in, feats):
        out, c = O.msa_branch_fwd(msa_in.numpy(), pair_in.numpy(), self.masks, self.P, i)
        return self.T(out), c

    def pair_branch_fwd(self, i, pair_mid, feats):
        out, c = O.pair_branch_fwd(pair_mid.numpy(), np.zeros_like(pair_mid.numpy()), self.masks,
                                   self.P, i, self.cfg)
        return self.T(out), c

    def loss(self, msa, pair):
        l, dm, dp = O.local_loss(self.cfg, msa.numpy(), pair.numpy())
        return torch.tensor([l], dtype=torch.float32), self.T(dm), self.T(dp)

    def msa_branch_bwd(self, i, d_msa, d_pair_acc, saved, feats):
        dm, dp = O.msa_branch_bwd(d_msa.numpy(), saved, self.P, i, self.grads)
        d_msa.copy_(self.T(dm))
        d_pair_acc.add_(self.T(dp))

    def opm_bwd_core(self, d, saved, prefix, feats):
        return self.T(O.opm_bwd(d.numpy(), saved, self.P, prefix, self.grads))

    def opm_ln_bwd(self, dxl, saved, prefix, d_msa):
        d_msa.add_(dxl)

    def pair_branch_bwd(self, i, d_pair, saved, feats):
        d_pair.copy_(self.T(O.pair_branch_bwd(d_pair.numpy(), saved, self.P, i, self.grads)))

    def embed_bwd(self, d_msa, d_pair, feats, rec, which="both"):
        O.embed_bwd(d_msa.numpy(), d_pair.numpy(), self.f, rec, self.grads)

    def forward_backward(self, feats, n_cycles=1, recompute=False):
        loss, grads, _ = O.serial_grads(self.cfg, self.P, self.f, n_cycles)
        self.grads = grads
        return torch.tensor([loss], dtype=torch.float32), None


def _worker(rank, world, port, mode, n_blocks, feat_seeds, out_path, n_cycles, recompute=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2207_05477_b200 import parallel as PL
    cfg = mini_cfg(n_blocks)
    grid = PL.GridConfig(dp=world) if mode == "dp" else PL.GridConfig.for_world(world)
    dpi, bpi, _ = grid.coords(rank)
    P = O.init_params(cfg, 7)
    feats = O.make_features(cfg, feat_seeds[dpi])
    eng = OracleEngine(cfg, P, feats)
    bp, world_comm = PL.build_groups(grid)
    if mode == "dp":
        loss = PL.dp_step(eng, feats, world_comm, grid, n_cycles=n_cycles, recompute=recompute)
    else:
        loss = PL.bp_step(eng, feats, bp, world_comm, grid, n_blocks, n_cycles=n_cycles,
                          recompute=recompute)
    if rank == 0:
        recs = [(r.group_axis, r.primitive, r.module, r.phase) for r in (bp.records if bp else [])]
        np.savez(out_path, loss=loss.numpy(), grads=eng.flat.numpy(),
                 recs=np.array(recs, dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, mode, n_blocks=2, feat_seeds=(3, 3), n_cycles=1, recompute=False):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r.npz")
        mp.spawn(_worker, args=(world, _free_port(), mode, n_blocks, list(feat_seeds), out, n_cycles,
                                recompute),
                 nprocs=world, join=True)
        r = np.load(out, allow_pickle=True)
        return float(r["loss"][0]), r["grads"], list(map(tuple, r["recs"]))


def _serial(n_blocks, feat_seed, n_cycles=1):
    cfg = mini_cfg(n_blocks)
    loss, grads, _ = O.serial_grads(cfg, O.init_params(cfg, 7), O.make_features(cfg, feat_seed),
                                    n_cycles)
    flat = np.concatenate([grads[n].ravel() for n, _, _ in O.param_specs(cfg)])
    return loss, flat


@pytest.mark.parametrize("world", [2, 4])
def test_bp_matches_serial(world):
    """bp2 and dp2 x bp2 (src/harness.py:392-616) == serial oracle, <= 1e-5."""
    loss, grads, recs = _run(world, "bp", feat_seeds=(3, 3))
    sl, sg = _serial(2, 3)
    assert abs(loss - sl) <= 1e-5
    assert np.abs(grads - sg).max() <= 1e-5


def test_bp_trace_three_broadcasts_one_allreduce_per_block():
    """tests/test_acceptance.py:156-166 of the reference."""
    from paper_2207_05477_b200 import planner
    _, _, recs = _run(2, "bp", n_blocks=1)
    assert planner.trace_counts([(r[2], r[1]) for r in recs]) == planner.expected_trace("bp", 1)
    block = [r for r in recs if r[2] in ("opm", "msa_stack", "pair_stack")]
    assert len(block) == 4
    assert sum(1 for r in block if r[1] == "broadcast") == 3
    assert sum(1 for r in block if r[1] == "allreduce") == 1


def test_dp_averages_over_replicas():
    """tests/test_harness.py:195-205 of the reference: DP grads == mean of serials."""
    loss, grads, _ = _run(2, "dp", n_blocks=1, feat_seeds=(3, 99))
    la, ga = _serial(1, 3)
    lb, gb = _serial(1, 99)
    assert abs(loss - (la + lb) / 2) <= 1e-6
    assert np.abs(grads - (ga + gb) / 2).max() <= 1e-6


def test_bp_with_recycling_matches_serial():
    loss, grads, _ = _run(2, "bp", n_blocks=1, n_cycles=2)
    sl, sg = _serial(1, 3, n_cycles=2)
    assert abs(loss - sl) <= 1e-5
    assert np.abs(grads - sg).max() <= 1e-5


def test_bp_recompute_bitwise_and_same_trace():
    """BP with per-branch recompute: each rank re-runs its own
    branch's forward from stored inputs; gradients are bitwise those of the
    stored-activation BP step and no collective is added."""
    l0, g0, r0 = _run(2, "bp", n_blocks=2)
    l1, g1, r1 = _run(2, "bp", n_blocks=2, recompute=True)
    assert l0 == l1 and np.array_equal(g0, g1)
    assert r0 == r1


def test_grid_config_rules():
    from paper_2207_05477_b200.parallel import GridConfig
    from paper_2207_05477_b200.errors import ContractError
    g = GridConfig(dp=2, bp=2)
    assert {g.coords(r) for r in range(g.world)} == {(0, 0, 0), (0, 1, 0), (1, 0, 0), (1, 1, 0)}
    assert GridConfig.for_world(8) == GridConfig(dp=4, bp=2)
    for bad in (dict(bp=3), dict(bp=2, dap=2), dict(dp=0)):
        with pytest.raises(ContractError):
            GridConfig(**bad)
    g = GridConfig(dp=2, dap=2)
    assert [g.coords(r) for r in range(4)] == [(0, 0, 0), (0, 0, 1), (1, 0, 0), (1, 0, 1)]


def test_recompute_plan_rules():
    """src/trainer.py:44-68: only the 'evoformer' stack recomputes."""
    from paper_2207_05477_b200.errors import ContractError
    from paper_2207_05477_b200.trainer import ExecutionPlan
    ExecutionPlan(recompute=("evoformer",)).validate()
    assert ExecutionPlan(recompute=("evoformer",)).recompute_on
    assert not ExecutionPlan().recompute_on
    with pytest.raises(ContractError):
        ExecutionPlan(recompute=("msa",)).validate()
    # extension over the reference (src/trainer.py:59-60): BP/DP plans recompute too
    ExecutionPlan(recompute=("evoformer",), dp=2, bp=2).validate()


def _dap_comm_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2207_05477_b200 import parallel as PL
    grid = PL.GridConfig(dap=world)
    dap, _ = PL.build_dap_groups(grid)
    rng = np.random.default_rng(rank)
    x = torch.from_numpy(rng.standard_normal((world * 3, 5)).astype(np.float32))
    ag = dap.allgather(x[:3], "msa_row_attn")
    rs = dap.reducescatter_sum(x, "opm")
    a2a = dap.alltoall(x, "tri_end")
    np.savez(out_path + f".{rank}", x=x.numpy(), ag=ag.numpy(), rs=rs.numpy(), a2a=a2a.numpy(),
             prims=np.array([r.primitive for r in dap.records]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_dap_comm_primitives_match_reference_semantics(world):
    """Comm.allgather / reducescatter_sum / alltoall on dim-0 chunks have the
    semantics of the reference's DapPar collectives (src/harness.py:262-293):
    concat of every rank's chunk, this rank's chunk of the sum, and chunk j to
    rank j landing rank-major."""
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "c")
        mp.spawn(_dap_comm_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        r = [dict(np.load(out + f".{k}.npz")) for k in range(world)]
    xs = [q["x"] for q in r]
    for k in range(world):
        assert np.array_equal(r[k]["ag"], np.concatenate([x[:3] for x in xs]))
        np.testing.assert_allclose(r[k]["rs"], sum(x[3 * k:3 * k + 3] for x in xs), rtol=1e-6)
        assert np.array_equal(r[k]["a2a"], np.concatenate([x[3 * k:3 * k + 3] for x in xs]))
        assert list(r[k]["prims"]) == ["allgather", "reducescatter", "alltoall"]


class _SlicedEngine:
    """Minimal engine for the bucketed gradient all-reduce: blocks own
    contiguous slices of a flat region, with a non-block head and tail."""

    spans = {0: (5, 12), 1: (12, 30), 2: (30, 31)}

    def __init__(self, g):
        self.g = g

    def block_grad_view(self, i):
        lo, hi = self.spans[i]
        return self.g[lo:hi], lo, hi


def _bucket_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2207_05477_b200 import parallel as PL
    _, world_comm = PL.build_groups(PL.GridConfig(dp=world))
    g = torch.arange(40, dtype=torch.float32) * (rank + 1)
    b = PL._GradBuckets(_SlicedEngine(g), world_comm)
    for i in (2, 1, 0):                      # backward order
        b.block_done(i)
    b.close(g)
    np.savez(out_path + f".{rank}", g=g.numpy(), prims=np.array([r.primitive for r in world_comm.records]),
             mods=np.array([r.module for r in world_comm.records]), nbytes=np.array([r.bytes for r in world_comm.records]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bucketed_grad_allreduce_sums_whole_region_one_record(world):
    """parallel._GradBuckets: per-block slices issued in backward order plus
    the uncovered head / tail at the close sum every element of the region
    over the world, and the trace holds one logical grad_sync all-reduce of
    the whole region (the reference's single collective, src/harness.py:607-616)."""
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "b")
        mp.spawn(_bucket_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        r = [dict(np.load(out + f".{k}.npz")) for k in range(world)]
    want = np.arange(40, dtype=np.float32) * sum(range(1, world + 1))
    for q in r:
        np.testing.assert_array_equal(q["g"], want)
        assert list(q["prims"]) == ["allreduce"] and list(q["mods"]) == ["grad_sync"]
        assert int(q["nbytes"][0]) == 40 * 4
