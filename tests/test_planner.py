"""Planner tables and plan (src/planner.py:37-193; the reference's
tests/test_planner.py and tests/test_acceptance.py:141-147)."""

import numpy as np
import torch

from paper_2207_05477_b200 import planner
from paper_2207_05477_b200.fusion import FusionEngine
from paper_2207_05477_b200.model import ModelConfig, flatten_params, init_params


def test_comm_tables_match_reference():
    assert planner.comm_total("dap", "full") == 24
    assert planner.comm_total("dap", "mini") == 16
    dap = planner.comm_counts("dap", "full")
    assert dap["msa_stack"] == {"alltoall": 4, "allgather": 1, "reducescatter": 1}
    assert dap["pair_stack"] == {"alltoall": 8, "allgather": 4, "reducescatter": 4}
    assert dap["opm"] == {"allgather": 1, "reducescatter": 1}
    bp = planner.comm_counts("bp")
    assert sum(n for m in bp.values() for n in m.values()) == 4
    assert planner.comm_counts("dp") == {}


def test_plan_matches_allocated_regions():
    cfg = ModelConfig(n_blocks=2, n_seq=8, n_res=16, c_m=32, c_z=16, heads=4, opm_dim=4)
    P = init_params(cfg, 7)
    st = FusionEngine([(n, P[n]) for n, _ in flatten_params(cfg)], device="cpu")
    held = sum(t.numel() * t.element_size() for t in st.regions.values())
    p = planner.plan(cfg, act_bytes=4)
    assert p["fused_region_bytes"] == held
    assert p["param_count"] == sum(int(np.prod(np.shape(P[n]))) for n, _ in flatten_params(cfg))
    assert p["launches_per_step"] == {"grad_sync": 1, "grad_clip": 2, "opt_update": 1, "ema": 1}
    r = planner.plan(cfg, recompute=True, act_bytes=2)
    assert r["recompute_saved_inputs_bytes"] == 2 * 2 * (8 * 16 * 32 + 16 * 16 * 16)
    assert planner.plan(cfg, dap=2)["comm_per_block_total"] == 16
    assert planner.plan(cfg, bp=2, dp=2)["grad_sync_collectives"] == 1
