"""Per-block collective tables and the memory / launch plan of a training step
(src/planner.py:37-193), for the trace-parity tests and the step reports.

Only the rows that describe this build's hot path are kept: the collective
counts of the BP and DAP blocks (checked against the recorded ``Comm``
traces), the fused optimizer's launches per step, and the byte counts of the
pooled parameter regions and of the recompute inputs (checked against the
allocator's measured peaks by ``memory_report``)."""

from __future__ import annotations

from collections import Counter

import numpy as np

# per-block collective counts (forward + backward), by stack.  "mini" is the
# block built here (triangle attention only); "full" adds both triangle
# multiplications (src/planner.py:41-50)
DAP_BLOCK_COUNTS_FULL = {
    "msa_stack": {"alltoall": 4, "allgather": 1, "reducescatter": 1},
    "pair_stack": {"alltoall": 8, "allgather": 4, "reducescatter": 4},
    "opm": {"allgather": 1, "reducescatter": 1},
}
DAP_BLOCK_COUNTS_MINI = {
    "msa_stack": {"alltoall": 4, "allgather": 1, "reducescatter": 1},
    "pair_stack": {"alltoall": 4, "allgather": 2, "reducescatter": 2},
    "opm": {"allgather": 1, "reducescatter": 1},
}
BP_BLOCK_COUNTS = {
    "msa_stack": {"broadcast": 1},
    "pair_stack": {"allreduce": 1, "broadcast": 1},
    "opm": {"broadcast": 1},
}
MODULE_STACK = {
    "msa_row_attn": "msa_stack", "msa_col_attn": "msa_stack",
    "tri_start": "pair_stack", "tri_end": "pair_stack",
    "opm": "opm", "msa_stack": "msa_stack", "pair_stack": "pair_stack",
}
FUSED_LAUNCHES = {"grad_sync": 1, "grad_clip": 2, "opt_update": 1, "ema": 1}


def comm_counts(axis: str, model: str = "mini") -> dict:
    """Per-block collective counts for one worker on ``axis`` ("dap" / "bp")."""
    if axis == "dap":
        table = DAP_BLOCK_COUNTS_FULL if model == "full" else DAP_BLOCK_COUNTS_MINI
    elif axis == "bp":
        table = BP_BLOCK_COUNTS
    else:
        return {}
    return {k: dict(v) for k, v in table.items()}


def comm_total(axis: str, model: str = "mini") -> int:
    return sum(n for mod in comm_counts(axis, model).values() for n in mod.values())


def trace_counts(records) -> Counter:
    """(stack, primitive) -> count over a ``Comm`` trace (block-level modules only)."""
    c = Counter()
    for r in records:
        stack = MODULE_STACK.get(r.module if hasattr(r, "module") else r[0])
        if stack:
            c[(stack, r.primitive if hasattr(r, "primitive") else r[1])] += 1
    return c


def expected_trace(axis: str, n_blocks: int, model: str = "mini") -> Counter:
    return Counter({(stack, prim): n * n_blocks
                    for stack, prims in comm_counts(axis, model).items() for prim, n in prims.items()})


def plan(cfg, dp: int = 1, bp: int = 1, dap: int = 1, recompute: bool = False,
         act_bytes: int = 2) -> dict:
    """src/planner.py:147-193 for this build.  Byte counts per worker."""
    from .fusion import REGIONS, build_layout, layout_total_bytes
    from .model import flatten_params
    named = list(flatten_params(cfg))
    shapes = [s for _, s in named]
    n_params = int(sum(int(np.prod(s)) if s else 1 for s in shapes))
    region = layout_total_bytes(build_layout(named))
    S, R = cfg.n_seq, cfg.n_res
    block_in = act_bytes * (S * R * cfg.c_m + R * R * cfg.c_z) // dap
    per_block = comm_counts("bp") if bp == 2 else comm_counts("dap") if dap > 1 else {}
    return {
        "comm_per_block": per_block,
        "comm_per_block_total": sum(n for m in per_block.values() for n in m.values()),
        # one all-reduce of the pooled grad region (+ the loss) closes every parallel step
        "grad_sync_collectives": 1 if dp * bp * dap > 1 else 0,
        "param_count": n_params,
        "param_slots": len(shapes),
        # the fp32 pooled regions (params, grads, Adam m / v, EMA) plus, in bf16,
        # the storage-dtype shadow the projections read (src/fusion.py layout)
        "fused_region_bytes": region * len(REGIONS) + (region // 2 if act_bytes == 2 else 0),
        "launches_per_step": dict(FUSED_LAUNCHES),
        "recompute_saved_inputs_bytes": cfg.n_blocks * block_in if recompute else 0,
        "act_bytes_per_el": act_bytes,
    }


def memory_report(planned: dict, measured_peak_bytes: int, static_bytes: int) -> dict:
    """Measured allocator peak of a step next to the plan's static terms."""
    return {
        "measured_peak_bytes": int(measured_peak_bytes),
        "static_bytes": int(static_bytes),
        "activation_peak_bytes": int(measured_peak_bytes - static_bytes),
        "planned_fused_region_bytes": planned["fused_region_bytes"],
        "planned_recompute_inputs_bytes": planned["recompute_saved_inputs_bytes"],
    }
