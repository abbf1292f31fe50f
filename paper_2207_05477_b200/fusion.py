"""Tensor fusion for the optimizer path, on the GPU (src/fusion.py).

All parameters live in one pooled fp32 region with 256-byte aligned slots
in the reference flatten order (``build_layout``, src/fusion.py:50-58), next
to equally laid-out grads / adam_m / adam_v / ema regions and, in bf16 mode,
a bf16 shadow of the params that the projections read.  The model writes
its gradients straight into the grad-region slots (no load/copy), and the
optimizer tail is three kernel launches over whole regions:
``evo_sumsq_f64`` (+ its finalize) and ``evo_adam_clip_ema``.
"""

from __future__ import annotations

from collections import Counter
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import ContractError

ALIGN = 256
REGIONS = ("params", "grads", "adam_m", "adam_v", "ema")


@dataclass
class OptimConfig:
    """src/fusion.py:31-38."""

    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    clip_norm: float = 0.1
    ema_decay: float = 0.999


@dataclass
class Slot:
    name: str
    shape: tuple
    offset: int  # bytes from region start
    nbytes: int
    padded_bytes: int


def build_layout(named_shapes, align: int = ALIGN) -> list:
    """Aligned slot table shared by all pooled regions (src/fusion.py:50-58)."""
    slots, off = [], 0
    for name, shape in named_shapes:
        nbytes = int(np.prod(shape, dtype=np.int64)) * 4 if shape else 4
        padded = -(-nbytes // align) * align
        slots.append(Slot(name, tuple(shape), off, nbytes, padded))
        off += padded
    return slots


def bias_correction_table(o: OptimConfig, max_len: int = 1 << 22) -> np.ndarray:
    """[2, T] fp32: np.float32(1 - beta**t) for t = 1..T (src/fusion.py:189-192),
    T the first step at which both corrections have rounded to exactly 1.0f
    (so the device's clamp at T is exact for every later step)."""
    rows = ([], [])
    t = 1
    while t <= max_len:
        b1 = np.float32(1.0 - o.beta1 ** t)
        b2 = np.float32(1.0 - o.beta2 ** t)
        rows[0].append(b1)
        rows[1].append(b2)
        if b1 == np.float32(1.0) and b2 == np.float32(1.0):
            break
        t += 1
    return np.array(rows, np.float32)


def layout_total_bytes(slots) -> int:
    return slots[-1].offset + slots[-1].padded_bytes if slots else 0


class LaunchCounter:
    """Per-phase launch tally with the reference's phases (src/fusion.py:65-77)."""

    PHASES = ("grad_sync", "grad_clip", "opt_update", "ema")

    def __init__(self):
        self.counts = Counter()

    def hit(self, phase: str, n: int = 1):
        if phase not in self.PHASES:
            raise ContractError(f"unknown launch phase {phase!r}")
        self.counts[phase] += n

    def total(self) -> int:
        return sum(self.counts.values())


class FusionEngine:
    """Owns the pooled parameter storage on the GPU and runs the optimizer
    tail (src/fusion.py:80-237, fused mode only -- the per-tensor mode exists
    in the reference to show what fusion removes)."""

    def __init__(self, named_params, optim: OptimConfig = None, device="cuda",
                 shadow_dtype=None, align: int = ALIGN):
        named_params = list(named_params)
        self.names = [n for n, _ in named_params]
        self.optim = optim or OptimConfig()
        self.launches = LaunchCounter()
        self.step_count = 0
        self.slots = build_layout([(n, np.shape(v)) for n, v in named_params], align)
        self._by_name = {s.name: s for s in self.slots}
        self.n_total = layout_total_bytes(self.slots) // 4
        host = np.zeros(self.n_total, np.float32)
        for (name, v), s in zip(named_params, self.slots):
            lo = s.offset // 4
            host[lo:lo + int(np.prod(s.shape, dtype=np.int64) or 1)] = np.asarray(v, np.float32).ravel()
        self.device = torch.device(device)
        self.regions = {r: torch.zeros(self.n_total, dtype=torch.float32, device=self.device)
                        for r in REGIONS}
        self.regions["params"].copy_(torch.from_numpy(host))
        self.regions["ema"].copy_(self.regions["params"])
        self.shadow = None
        if shadow_dtype is not None and shadow_dtype != torch.float32:
            self.shadow = torch.empty(self.n_total, dtype=shadow_dtype, device=self.device)
            ops.cast(self.regions["params"], self.shadow)
        self.sumsq = torch.zeros(1, dtype=torch.float64, device=self.device)
        # Adam's step counter t on the device (advanced by the sumsq kernel), so
        # a CUDA graph that captured step() replays with the right t; the
        # bias corrections are tabulated once with the reference's expression
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.bc_table = torch.from_numpy(bias_correction_table(self.optim)).to(self.device)
        self.bc = torch.ones(2, dtype=torch.float32, device=self.device)
        self._views = {}

    # -- storage access --------------------------------------------------------

    def _view(self, buf: torch.Tensor, name: str) -> torch.Tensor:
        s = self._by_name[name]
        lo = s.offset // 4
        n = int(np.prod(s.shape, dtype=np.int64)) if s.shape else 1
        return buf[lo:lo + n].view(s.shape if s.shape else (1,))

    def view(self, region: str, name: str) -> torch.Tensor:
        key = (region, name)
        v = self._views.get(key)
        if v is None:
            buf = self.shadow if region == "shadow" else self.regions[region]
            v = self._views[key] = self._view(buf, name)
        return v

    def param(self, name):
        return self.view("params", name)

    def grad(self, name):
        return self.view("grads", name)

    def weight(self, name):
        """The projection operand: the bf16 shadow in bf16 mode, else the fp32 param."""
        return self.view("shadow" if self.shadow is not None else "params", name)

    def zero_grads(self):
        self.regions["grads"].zero_()

    def load_grads(self, grads: dict):
        missing = [n for n in self.names if n not in grads]
        if missing:
            raise ContractError(f"missing gradients for {missing[:3]}...")
        for n in self.names:
            g = grads[n]
            g = g if isinstance(g, torch.Tensor) else torch.from_numpy(np.asarray(g, np.float32))
            self.grad(n).copy_(g.reshape(self.grad(n).shape))

    def layout_rows(self) -> list:
        rows = []
        for region in REGIONS:
            for s in self.slots:
                rows.append({"name": s.name, "shape": "x".join(map(str, s.shape)) or "1",
                             "region": region, "offset": s.offset, "padded_bytes": s.padded_bytes})
        return rows

    # -- optimizer tail ----------------------------------------------------------

    def grad_sync(self, reducer=None):
        """``reducer(region) -> None`` reduces the whole grad region in place
        (one collective, e.g. NCCL all-reduce average)."""
        self.launches.hit("grad_sync", 1)
        if reducer is not None:
            reducer(self.regions["grads"])

    def step(self):
        """clip + Adam + EMA over the pooled regions; returns the fp64
        sum-of-squares of the pre-clip gradient as a device tensor.  The step
        counter advances on the device (``step_dev``), so this sequence can be
        captured in a CUDA graph; ``note_replayed_step`` keeps the host count."""
        o = self.optim
        self.step_count += 1
        f32 = np.float32
        ops.sumsq_f64_step(self.regions["grads"], self.sumsq, self.step_dev, self.bc_table, self.bc)
        self.launches.hit("grad_clip", 2)
        r = self.regions
        ops.adam_clip_ema_dev(r["params"], r["grads"], r["adam_m"], r["adam_v"], r["ema"], self.shadow,
                              self.sumsq, float(o.clip_norm), float(f32(o.lr)), float(f32(o.beta1)),
                              float(f32(1 - o.beta1)), float(f32(o.beta2)), float(f32(1 - o.beta2)),
                              float(f32(o.eps)), self.bc, float(f32(o.ema_decay)),
                              float(f32(1.0) - f32(o.ema_decay)))
        self.launches.hit("opt_update", 1)
        self.launches.hit("ema", 1)
        return self.sumsq

    def note_replayed_step(self):
        """A captured step() was replayed: advance the host-side counters the
        way step() itself would have."""
        self.step_count += 1
        self.launches.hit("grad_clip", 2)
        self.launches.hit("opt_update", 1)
        self.launches.hit("ema", 1)

    def device_step_count(self) -> int:
        return int(self.step_dev.item())

    def apply(self, grads: dict = None, reducer=None, sync: bool = True):
        """Full optimizer tail (src/fusion.py:226-233); returns the pre-clip
        global gradient norm (host float when ``sync``)."""
        if grads is not None:
            self.load_grads(grads)
        self.grad_sync(reducer)
        sq = self.step()
        return float(np.sqrt(sq.item())) if sync else sq

    def params_snapshot(self) -> dict:
        return {n: self.param(n).detach().cpu().numpy().copy() for n in self.names}
