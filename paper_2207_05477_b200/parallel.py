"""Branch Parallelism (BP) and data parallelism (DP) over torch.distributed.

Rebuilds the reference's grid runner (src/harness.py:53-76, 392-553,
570-645) with one process per GPU (NCCL over NVLink/NVSwitch; gloo for the
CPU tests) instead of thread-simulated ranks:

* rank = dp_i * bp + bp_i (``GridConfig.rank`` with dap = 1);
* BP pairs {2k, 2k+1}: bp rank 0 runs the MSA stack (row + column attention,
  MSA transition) and the outer-product mean, bp rank 1 runs the pair stack
  (triangle attention start/end, pair transition [, TriangleMultiplication]);
  the two branches of a block are independent given the block inputs
  because the OPM reads the block-input MSA (src/model.py:440), so rank 1's
  pair stack of block i overlaps rank 0's MSA stack of block i;
* per block and step: forward broadcasts opm (root 0), msa' (root 0),
  pair' (root 1); backward one all-reduce of d(pair_in) -- exactly the
  reference's 3 Broadcast + 1 AllReduce (tests/test_acceptance.py:156-166);
* forward broadcasts are asynchronous on NCCL: each rank's stream waits only
  where it reads a received tensor, so rank 0 computes opm(i+1) while rank 1
  still runs the pair stack of block i;
* gradient exchange: the closing broadcast of d(msa) (module "msa_grad"),
  then the all-reduce of the pooled grad region over the world (each
  parameter's gradient is non-zero on exactly one rank of a BP pair, so the
  sum equals the reference's per-branch broadcasts), scaled by 1/dp -- the
  DP average of src/harness.py:607-616 folded into the same collective.  It
  is bucketed per block and issued as each block's backward finishes
  (``_GradBuckets``), one logical trace record.

The step is written against a small engine protocol (``BlockEngine`` on the
GPU; the tests drive it with an adapter around the CPU oracle), and a
``Comm`` wrapper that records the reference's CommRecord trace
(src/harness.py:79-101).
"""

from __future__ import annotations

import csv
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from .errors import ContractError


@dataclass(frozen=True)
class GridConfig:
    """src/harness.py:53-76.  bp and dap do not compose; dp composes with either
    (ranks: dp outermost, then bp, then dap)."""

    dp: int = 1
    bp: int = 1
    dap: int = 1

    def __post_init__(self):
        if self.dp < 1 or self.bp < 1 or self.dap < 1:
            raise ContractError("grid axes must be >= 1")
        if self.bp not in (1, 2):
            raise ContractError("branch parallelism supports size 1 or 2")
        if self.bp > 1 and self.dap > 1:
            raise ContractError("bp and dap axes do not compose")

    @property
    def world(self) -> int:
        return self.dp * self.bp * self.dap

    def coords(self, rank: int):
        inner = self.bp * self.dap
        return rank // inner, (rank % inner) // self.dap, rank % self.dap

    def rank(self, dpi: int, bpi: int, dapi: int = 0) -> int:
        return dpi * self.bp * self.dap + bpi * self.dap + dapi

    @staticmethod
    def for_world(world: int) -> "GridConfig":
        """1 -> serial, 2 -> bp2, 2k -> dp k x bp 2 (the survey's grids)."""
        if world == 1:
            return GridConfig()
        if world % 2:
            return GridConfig(dp=world)
        return GridConfig(dp=world // 2, bp=2)


@dataclass
class CommRecord:
    step: int
    phase: str
    group_axis: str
    group_id: int
    seq: int
    primitive: str
    bytes: int
    module: str


CSV_COLUMNS = ["step", "phase", "group_axis", "group_id", "seq", "primitive", "bytes", "module"]


def dump_comm_csv(records, path):
    """Same columns as the reference trace (src/harness.py:91-101)."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_COLUMNS)
        for r in records:
            w.writerow([r.step, r.phase, r.group_axis, r.group_id, r.seq, r.primitive, r.bytes,
                        r.module])


class Comm:
    """One rank's endpoint on one grid axis, over a torch.distributed group."""

    def __init__(self, axis: str, group_id: int, ranks: list, group=None):
        self.axis = axis
        self.group_id = group_id
        self.ranks = list(ranks)
        self.group = group
        self.size = len(ranks)
        self.rank = self.ranks.index(dist.get_rank()) if dist.is_initialized() else 0
        self._seq = 0
        self.records: list = []
        self.step = 0
        self.phase = "fwd"

    def _rec(self, primitive, t, module):
        self.records.append(CommRecord(self.step, self.phase, self.axis, self.group_id, self._seq,
                                       primitive, t.numel() * t.element_size(), module))
        self._seq += 1

    def broadcast(self, t: torch.Tensor, root: int, module: str, async_op: bool = False):
        """In place: ``t`` is the payload on the root, the receive buffer elsewhere.

        ``async_op`` (device tensors on NCCL): the collective is ordered after
        the work already queued on the current stream but the stream does not
        wait for it; returns a handle whose ``wait()`` makes the current stream
        wait (None when the collective already completed, e.g. on gloo)."""
        handle = None
        if self._host(t):
            h = t.cpu()
            dist.broadcast(h, src=self.ranks[root], group=self.group)
            t.copy_(h)
        elif async_op and self._nccl(t):
            handle = dist.broadcast(t, src=self.ranks[root], group=self.group, async_op=True)
        else:
            dist.broadcast(t, src=self.ranks[root], group=self.group)
        self._rec("broadcast", t, module)
        return handle if async_op else t

    def allreduce_sum(self, t: torch.Tensor, module: str) -> torch.Tensor:
        self.allreduce_sum_raw(t)
        self._rec("allreduce", t, module)
        return t

    def allreduce_sum_raw(self, t: torch.Tensor, stream=None, async_op: bool = False):
        """Sum over the group without a trace record (one bucket of a logical
        collective that the caller records once).  With ``stream`` the
        collective is ordered after that stream's queued work; with
        ``async_op`` on NCCL the handle is returned (see ``broadcast``)."""
        ctx = torch.cuda.stream(stream) if stream is not None else _NullCtx()
        with ctx:
            if self._host(t):
                h = t.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
                t.copy_(h)
            elif async_op and self._nccl(t):
                return dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return None

    def _nccl(self, t):
        return t.is_cuda and dist.get_backend(self.group) == "nccl"

    # -- DAP primitives (src/harness.py:262-293): dim-0 chunk i <-> group rank i ----
    # NCCL runs them on device buffers; a gloo group (the CPU tests, and the
    # several-ranks-on-one-GPU GPU test) gets host copies, and its missing
    # reduce-scatter is an all-reduce plus this rank's chunk.

    def _host(self, t):
        return t.is_cuda and dist.get_backend(self.group) == "gloo"

    def allgather(self, t: torch.Tensor, module: str) -> torch.Tensor:
        """[n, ...] per rank -> [size * n, ...], rank-major."""
        t = t.contiguous()
        out = torch.empty((self.size * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        if self._host(t):
            parts = [torch.empty_like(t, device="cpu") for _ in range(self.size)]
            dist.all_gather(parts, t.cpu(), group=self.group)
            out.copy_(torch.cat(parts))
        else:
            dist.all_gather_into_tensor(out, t, group=self.group)
        self._rec("allgather", t, module)
        return out

    def reducescatter_sum(self, t: torch.Tensor, module: str) -> torch.Tensor:
        """[size * n, ...] per rank -> [n, ...]: chunk ``rank`` summed over ranks."""
        t = t.contiguous()
        n = t.shape[0] // self.size
        if n * self.size != t.shape[0]:
            raise ContractError(f"cannot scatter extent {t.shape[0]} over {self.size} workers")
        if self._host(t) or (not t.is_cuda and dist.get_backend(self.group) == "gloo"):
            h = t.cpu() if t.is_cuda else t.clone()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            out = h[self.rank * n:(self.rank + 1) * n].to(t.device).contiguous()
        else:
            out = torch.empty((n,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            dist.reduce_scatter_tensor(out, t, op=dist.ReduceOp.SUM, group=self.group)
        self._rec("reducescatter", t, module)
        return out

    def alltoall(self, t: torch.Tensor, module: str, out: torch.Tensor = None) -> torch.Tensor:
        """Chunk j of dim 0 goes to rank j; received chunks land rank-major."""
        t = t.contiguous()
        if t.shape[0] % self.size:
            raise ContractError(f"cannot split extent {t.shape[0]} over {self.size} workers")
        out = torch.empty_like(t) if out is None else out
        if self._host(t):
            h = torch.empty_like(t, device="cpu")
            dist.all_to_all_single(h, t.cpu(), group=self.group)
            out.copy_(h)
        else:
            dist.all_to_all_single(out, t, group=self.group)
        self._rec("alltoall", t, module)
        return out


def build_groups(grid: GridConfig):
    """All ranks must create every group in the same order (torch.distributed
    rule).  Returns (bp Comm or None, world Comm)."""
    me = dist.get_rank()
    dpi, bpi, _ = grid.coords(me)
    bp_comm = None
    if grid.bp == 2:
        for d in range(grid.dp):
            ranks = [grid.rank(d, 0), grid.rank(d, 1)]
            g = dist.new_group(ranks)
            if d == dpi:
                bp_comm = Comm("bp", d, ranks, g)
    world = Comm("dp", 0, list(range(grid.world)), None)
    return bp_comm, world


def build_dap_groups(grid: GridConfig):
    """Returns (dap Comm of this rank, world Comm); every rank creates every group."""
    me = dist.get_rank()
    dpi = grid.coords(me)[0]
    dap_comm = None
    for d in range(grid.dp):
        ranks = [grid.rank(d, 0, j) for j in range(grid.dap)]
        g = dist.new_group(ranks)
        if d == dpi:
            dap_comm = Comm("dap", d, ranks, g)
    return dap_comm, Comm("dp", 0, list(range(grid.world)), None)


@dataclass
class StepResult:
    loss: float
    records: list = field(default_factory=list)


def bp_step(engine, feats, bp: Comm, world: Comm, grid: GridConfig, n_blocks: int,
            step: int = 0, n_cycles: int = 1, recompute: bool = False):
    """One branch-parallel forward/backward (src/harness.py:392-553) plus the
    fused gradient all-reduce.  Returns the device loss tensor ([1]); the
    pooled grad region ends up holding the world-averaged gradients.

    ``recompute`` (the reference restricts recompute_grads to one
    worker, src/trainer.py:59-60): each rank keeps only its own branch's
    block inputs -- (msa, pair) on rank 0, pair_mid on rank 1 -- and re-runs
    its branch forward right before the block's backward.  Both branches'
    forwards need only local inputs, so recompute adds no collective and the
    comm trace is unchanged."""
    me = bp.rank
    for c in (bp, world):
        c.step = step
        c.phase = "fwd"
    refresh = getattr(engine, "refresh_weights", None)
    if refresh is not None:
        refresh()
    engine.zero_grads()
    prev = None
    for _ in range(max(0, n_cycles - 1)):  # replicated recycling warm-up, no comm (:406-415)
        prev = engine.forward_only(feats, prev)
    msa, pair, rec = engine.embed_fwd(feats, prev)
    saved = []
    # Forward, per block i: broadcasts opm(i) (root 0), msa(i) (root 0),
    # pair(i) (root 1) in that order on both ranks.  On NCCL they are issued
    # asynchronously and each rank's stream waits only where it reads a
    # received tensor, so rank 0 computes opm(i+1) (it needs only msa(i))
    # while rank 1's pair stack of block i still runs, and rank 1 posts the
    # msa(i) receive before its pair stack instead of stalling on it.
    if me == 0:
        h_pair = None
        opm, so = (engine.opm_fwd(msa, "block0.opm", feats, pair_res=None) if n_blocks else (None, None))
        if n_blocks:
            bp.broadcast(opm, 0, "opm", async_op=True)
        for i in range(n_blocks):
            _wait(h_pair)                                # pair(i-1) from rank 1
            msa_out, sm = engine.msa_branch_fwd(i, msa, pair, feats)
            bp.broadcast(msa_out, 0, "msa_stack", async_op=True)
            pair_out = engine.empty_like(pair)
            h_pair = bp.broadcast(pair_out, 1, "pair_stack", async_op=True)
            saved.append((msa, pair) if recompute else (so, sm))
            if i + 1 < n_blocks:
                opm, so = engine.opm_fwd(msa_out, f"block{i + 1}.opm", feats, pair_res=None)
                bp.broadcast(opm, 0, "opm", async_op=True)
            msa, pair = msa_out, pair_out
        _wait(h_pair)
    else:
        h_msa = h_opm = None
        opm = None
        if n_blocks:
            opm = engine.empty_like(pair)
            h_opm = bp.broadcast(opm, 0, "opm", async_op=True)
        for i in range(n_blocks):
            msa_out = engine.empty_like(msa)
            h_msa = bp.broadcast(msa_out, 0, "msa_stack", async_op=True)
            _wait(h_opm)
            pair_mid = engine.add(pair, opm)
            pair_out, sp = engine.pair_branch_fwd(i, pair_mid, feats)
            bp.broadcast(pair_out, 1, "pair_stack", async_op=True)
            saved.append(pair_mid if recompute else sp)
            if i + 1 < n_blocks:
                opm = engine.empty_like(pair)
                h_opm = bp.broadcast(opm, 0, "opm", async_op=True)
            msa, pair = msa_out, pair_out
        _wait(h_msa)
    opm = None
    loss, d_msa, d_pair = engine.loss(msa, pair)

    for c in (bp, world):
        c.phase = "bwd"
    deferred = getattr(engine, "deferred", None)
    buckets = _GradBuckets(engine, world)
    for i in reversed(range(n_blocks)):
        if recompute and me == 0:
            msa_in, pair_in = saved[i]
            so = engine.opm_fwd(msa_in, f"block{i}.opm", feats, pair_res=None)[1]
            sm = engine.msa_branch_fwd(i, msa_in, pair_in, feats)[1]
            saved[i] = (so, sm)
        elif recompute:
            saved[i] = engine.pair_branch_fwd(i, saved[i], feats)[1]
        ctx = deferred() if deferred is not None else _NullCtx()
        with ctx:
            _bp_block_bwd(engine, feats, bp, me, i, saved, d_msa, d_pair)
            if me == 0:
                d_pair = saved[i]  # the all-reduced d(pair_in), see _bp_block_bwd
        buckets.block_done(i)      # block i's gradients are final on this rank
        saved[i] = None
    # embeddings: each worker closes out its own branch (src/harness.py:518-522)
    if me == 0:
        engine.embed_bwd(d_msa, engine.zeros_like(d_pair), feats, rec, which="msa")
    else:
        engine.embed_bwd(engine.zeros_like(d_msa), d_pair, feats, rec, which="pair")
    return _bp_close(engine, bp, world, grid, me, d_msa, loss, buckets)


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def _wait(handle):
    if handle is not None:
        handle.wait()


class _GradBuckets:
    """The world gradient all-reduce, bucketed per Evoformer block.

    The reference sums the flattened gradients of every parameter in one
    collective after the backward (src/harness.py:607-616).  Here block i's
    slice of the pooled grad region is all-reduced as soon as block i's
    backward has produced it -- asynchronously on NCCL, ordered after the
    stream that finished it -- so it overlaps the backward of blocks i-1 .. 0;
    the rest of the region (embeddings, recycling) goes at the close.  The
    trace keeps the reference's single logical "grad_sync" record (bytes of
    the whole region).  Engines without ``block_grad_view`` (the CPU oracle
    adapter) fall back to the one-shot collective."""

    def __init__(self, engine, world):
        self.view = getattr(engine, "block_grad_view", None)
        self.world = world
        self.handles = []
        self.done = []  # (lo, hi) element ranges already issued

    def block_done(self, i, stream=None):
        if self.view is None:
            return
        v, lo, hi = self.view(i)
        self.handles.append(self.world.allreduce_sum_raw(v, stream=stream, async_op=True))
        self.done.append((lo, hi))

    def close(self, g):
        """All-reduce what is left of ``g``, wait for every bucket, record once."""
        if self.view is None:
            self.world.allreduce_sum(g, "grad_sync")
            return
        cur = 0
        for lo, hi in sorted(self.done):
            if lo > cur:
                self.handles.append(self.world.allreduce_sum_raw(g[cur:lo], async_op=True))
            cur = max(cur, hi)
        if cur < g.numel():
            self.handles.append(self.world.allreduce_sum_raw(g[cur:], async_op=True))
        for h in self.handles:
            _wait(h)
        self.handles.clear()
        self.world._rec("allreduce", g, "grad_sync")


def _bp_block_bwd(engine, feats, bp, me, i, saved, d_msa, d_pair):
    """Block i backward on this BP rank (src/harness.py:497-516).  Rank 0
    leaves the all-reduced d(pair_in) in saved[i] (its input d_pair is not
    updated in place); rank 1 updates d_pair in place."""
    if me == 0:
        so, sm = saved[i]
        b_contrib = engine.zeros_like(d_pair)
        engine.msa_branch_bwd(i, d_msa, b_contrib, sm, feats)       # d_msa -> d(msa_in) part
        s = b_contrib.clone()
        bp.allreduce_sum(s, "pair_stack")
        d_opm = s - b_contrib                                       # src/harness.py:505
        dxl = engine.opm_bwd_core(d_opm, so, f"block{i}.opm", feats)
        engine.opm_ln_bwd(dxl, so, f"block{i}.opm", d_msa)
        saved[i] = s
    else:
        engine.pair_branch_bwd(i, d_pair, saved[i], feats)         # d_pair -> d(pair_mid)
        bp.allreduce_sum(d_pair, "pair_stack")


def _bp_close(engine, bp, world, grid, me, d_msa, loss, buckets=None):
    for c in (bp, world):
        c.phase = "grad-sync"
    closing = d_msa if me == 0 else engine.empty_like(d_msa)
    bp.broadcast(closing, 0, "msa_grad")
    g = engine.grad_region()
    (buckets or _GradBuckets(None, world)).close(g)
    if grid.dp > 1:
        g.mul_(np.float32(1.0 / grid.dp).item())
    lt = loss.reshape(1).clone()
    if grid.dp > 1:
        # every rank of a BP pair holds the same replicated loss: world sum / world
        world.allreduce_sum(lt, "loss")
        lt.mul_(np.float32(1.0 / grid.world).item())
    return lt


def dp_step(engine, feats, world: Comm, grid: GridConfig, n_cycles: int = 1, step: int = 0,
            recompute: bool = False):
    """Pure data parallelism: serial fwd+bwd per replica, one all-reduce of the
    pooled grad region (src/harness.py:607-616)."""
    world.step = step
    world.phase = "grad-sync"
    buckets = _GradBuckets(engine, world)
    if buckets.view is not None:
        loss, _ = engine.forward_backward(feats, n_cycles, recompute=recompute, grad_ready=buckets.block_done)
    else:
        loss, _ = engine.forward_backward(feats, n_cycles, recompute=recompute)
    g = engine.grad_region()
    buckets.close(g)
    g.mul_(np.float32(1.0 / grid.dp).item())
    lt = loss.reshape(1).clone()
    world.allreduce_sum(lt, "loss")
    lt.mul_(np.float32(1.0 / grid.dp).item())
    return lt
