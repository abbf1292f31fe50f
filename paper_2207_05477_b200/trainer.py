"""Training-step orchestration (src/trainer.py) on the GPU engine.

One step: draw recycles (or pin them), build the step's synthetic features
(src/trainer.py:98-101, src/model.py:274-288), copy them host->device, run
forward + hand-written backward with gradients landing in the pooled grad
region, then the fused optimizer tail (clip + Adam + EMA).  The whole
device-side step can be captured into one CUDA graph (``capture()``): the
feature buffers keep fixed device addresses and are refreshed in place.
"""

from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .engine import BlockEngine, DeviceFeatures
from .errors import ContractError, TrainingAborted
from .fusion import FusionEngine, OptimConfig
from .model import (ModelConfig, draw_num_recycles, flatten_params, init_params,
                    make_features, step_feature_seed)


@dataclass
class ExecutionPlan:
    """src/trainer.py:37-79 (single-worker part; BP/DP in parallel.py)."""

    dp: int = 1
    bp: int = 1
    dap: int = 1
    fuse_ops: bool = True
    fuse_tensors: bool = True
    recompute: tuple = ()  # subset of {"evoformer"}
    act_dtype: str = "bf16"
    chunk: int = 0
    seed: int = 32
    steps: int = 10
    fixed_recycles: int = 0  # >0 pins n_recycles (throughput runs use 1)

    def validate(self):
        if self.dp < 1 or self.bp not in (1, 2) or self.dap < 1:
            raise ContractError("supported grids: dp>=1, bp in {1,2}, dap>=1")
        if self.bp > 1 and self.dap > 1:
            raise ContractError("plan.bp: bp and dap axes do not compose")
        if self.act_dtype not in ("f32", "bf16"):
            raise ContractError(f"act_dtype must be f32 or bf16, got {self.act_dtype!r}")
        if self.chunk < 0:
            raise ContractError("chunk must be >= 0")
        unknown = set(self.recompute) - {"evoformer"}
        if unknown:
            raise ContractError(f"unknown recompute stacks {sorted(unknown)}")

    @property
    def recompute_on(self) -> bool:
        return "evoformer" in self.recompute

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.act_dtype == "bf16" else torch.float32


class PinnedFeatures:
    """Host staging of one step's features in pinned memory."""

    def __init__(self, cfg: ModelConfig):
        S, R, F = cfg.n_seq, cfg.n_res, cfg.feat_dim
        self.msa_feat = torch.empty((S * R, F), dtype=torch.float32).pin_memory()
        self.pair_feat = torch.empty((R * R, F), dtype=torch.float32).pin_memory()
        self.msa_mask = torch.empty((S * R,), dtype=torch.float32).pin_memory()
        self.pair_mask = torch.empty((R * R,), dtype=torch.float32).pin_memory()

    def fill(self, feats):
        for k in ("msa_feat", "pair_feat", "msa_mask", "pair_mask"):
            getattr(self, k).copy_(torch.from_numpy(
                np.ascontiguousarray(getattr(feats, k), np.float32).reshape(getattr(self, k).shape)))

    @property
    def nbytes(self) -> int:
        return sum(getattr(self, k).numel() * 4 for k in ("msa_feat", "pair_feat", "msa_mask", "pair_mask"))


@dataclass
class Trainer:
    cfg: ModelConfig
    plan: ExecutionPlan
    store: FusionEngine
    engine: BlockEngine
    feats: DeviceFeatures
    host: PinnedFeatures
    history: list = field(default_factory=list)
    graph: object = None
    graph_loss: object = None

    @classmethod
    def create(cls, cfg: ModelConfig, plan: ExecutionPlan, optim: OptimConfig = None,
               device="cuda", params: dict = None):
        plan.validate()
        cfg.validate()
        params = params if params is not None else init_params(cfg, plan.seed)
        named = [(n, params[n]) for n, _ in flatten_params(cfg)]
        store = FusionEngine(named, optim or OptimConfig(), device=device,
                             shadow_dtype=plan.torch_dtype)
        engine = BlockEngine(cfg, store, plan.torch_dtype)
        f0 = make_features(cfg, step_feature_seed(plan.seed, 0))
        feats = DeviceFeatures(f0, device, cfg)
        host = PinnedFeatures(cfg)
        return cls(cfg, plan, store, engine, feats, host)

    def n_recycles(self, step: int) -> int:
        if self.plan.fixed_recycles:
            return self.plan.fixed_recycles
        return draw_num_recycles(self.plan.seed, step)

    def stage_features(self, step: int, feats=None):
        """Host-side feature generation for ``step`` into pinned memory."""
        feats = feats or make_features(self.cfg, step_feature_seed(self.plan.seed, step))
        self.host.fill(feats)

    def attach_parallel(self, step_fn, comms):
        """Route ``device_step`` through a multi-rank step -- ``step_fn(engine,
        feats, n_cycles, step)`` returning the device loss after the gradient
        exchange (parallel.bp_step / dp_step, dap.dap_step) -- and count the
        CommRecords its ``comms`` endpoints log as the step's ``comm_records``
        (src/trainer.py:192-247, src/harness.py:79-101)."""
        self.parallel_step = step_fn
        self.comms = list(comms)

    def comm_records(self):
        """Every CommRecord logged so far, all endpoints (dump with
        parallel.dump_comm_csv)."""
        return [r for c in getattr(self, "comms", ()) for r in c.records]

    def device_step(self, n_cycles: int, h2d: bool = True, step: int = 0):
        """H2D of the staged features (unless ``h2d`` is False: the features
        already in HBM are used), fwd+bwd, optimizer; returns the device loss
        tensor (no host sync)."""
        if h2d:
            self.feats.copy_from_host(self.host)
        par = getattr(self, "parallel_step", None)
        if par is not None:   # the step's own collective already synced the grad region
            loss = par(self.engine, self.feats, n_cycles, step)
        else:
            loss, _ = self.engine.forward_backward(self.feats, n_cycles,
                                                   recompute=self.plan.recompute_on)
        self.store.grad_sync(None)
        self.store.step()
        return loss

    def capture(self, n_cycles: int = 1, warmup: int = 2):
        """Capture the device part of ``device_step`` (fwd+bwd+optimizer on the
        features resident in ``self.feats``) into a CUDA graph, after eager
        warm-up.  ``replay(host)`` copies a step's features in first."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.device_step(n_cycles, h2d=False)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        count = self.store.step_count
        with torch.cuda.graph(g):
            self.graph_loss = self.device_step(n_cycles, h2d=False)
        self.store.step_count = count     # capture records the step, it does not run it
        self.graph = g
        return g

    def replay(self, host: "PinnedFeatures" = None):
        """One captured device step; with ``host`` (pinned features) their H2D
        copy is enqueued first, else the features already in HBM are used.
        Returns the device loss tensor.  Adam's step counter advances on the
        device, so replayed steps equal eager ones."""
        if host is not None:
            self.feats.copy_from_host(host)
        self.graph.replay()
        self.store.note_replayed_step()
        return self.graph_loss

    def train_step(self, step: int):
        """src/trainer.py:192-247 (serial): returns (loss, metrics).  Metric keys
        follow the reference: ``launches`` are this step's optimizer-phase
        launches (src/fusion.py:65-77), ``op_count`` this step's launches of the
        library's own kernels, ``ledger_peak_bytes`` the device-memory peak of
        the step above what was live before it (the reference's ledger peak)."""
        from . import _lib
        n_rec = self.n_recycles(step)
        self.stage_features(step)
        launches_before = dict(self.store.launches.counts)
        ops_before = _lib.launch_count()
        dev = torch.device(self.store.device)
        live_before = torch.cuda.memory_allocated(dev)
        torch.cuda.reset_peak_memory_stats(dev)
        recs_before = len(self.comm_records())
        loss_t = self.device_step(n_rec, step=step)
        loss = float(loss_t.item())
        if not math.isfinite(loss):
            raise TrainingAborted(step, f"non-finite loss {loss!r}")
        grad_norm = float(np.sqrt(self.store.sumsq.item()))
        launches = {k: self.store.launches.counts[k] - launches_before.get(k, 0)
                    for k in self.store.launches.PHASES}
        metrics = {"step": step, "loss": loss, "grad_norm": grad_norm, "n_recycles": n_rec,
                   "launches": launches, "comm_records": len(self.comm_records()) - recs_before,
                   "ledger_peak_bytes": int(torch.cuda.max_memory_allocated(dev) - live_before),
                   "op_count": int(_lib.launch_count() - ops_before),
                   "blocks_executed": self.cfg.n_blocks * n_rec}
        self.history.append(metrics)
        return loss, metrics

    def train_loop(self, steps: int, metrics_path=None):
        """src/trainer.py:250-262: ``steps`` steps, one compact JSON line of
        metrics per step into ``metrics_path`` (metrics.jsonl)."""
        fh = open(metrics_path, "w") if metrics_path else None
        losses = []
        try:
            for s in range(steps):
                loss, metrics = self.train_step(s)
                losses.append(loss)
                if fh:
                    fh.write(json.dumps(metrics, separators=(",", ":")) + "\n")
        finally:
            if fh:
                fh.close()
        return losses

    def bench_protocol(self, total: int = 105, discard: int = 5, _spike=None):
        """src/trainer.py:269-303: run ``total`` steps, drop the first
        ``discard`` and average the counters and step times of the rest
        (bench.json).  ``_spike`` = (step, key, amount) perturbs one step's
        counters so tests can show discarded steps do not leak in."""
        if total <= discard:
            raise ContractError("total must exceed the discarded prefix")
        per_step, times = [], []
        t0 = time.perf_counter()
        for s in range(total):
            s0 = time.perf_counter()
            _, metrics = self.train_step(s)
            times.append(time.perf_counter() - s0)
            metrics = dict(metrics)
            metrics["launch_total"] = sum(metrics["launches"].values())
            if _spike is not None and s == _spike[0]:
                metrics[_spike[1]] = metrics.get(_spike[1], 0) + _spike[2]
            per_step.append(metrics)
        wall = time.perf_counter() - t0
        kept, kept_t = per_step[discard:], times[discard:]
        counters = {k: float(np.mean([m[k] for m in kept])) for k in COUNTER_KEYS + ("launch_total",)}
        return {"total_steps": total, "discarded": discard, "averaged_steps": len(kept),
                "counters": counters, "mean_step_seconds": float(np.mean(kept_t)),
                "steps_per_second": float(1.0 / np.mean(kept_t)), "wall_seconds": wall,
                "seed": self.plan.seed}


COUNTER_KEYS = ("loss", "grad_norm", "n_recycles", "comm_records", "ledger_peak_bytes", "op_count")
