"""Training-step time and peak HBM at a named shape, with or without
per-block recompute (src/trainer.py:108-179).

    python tools/time_shape.py --shape F --blocks 48 --recompute
    python tools/time_shape.py --shape I --blocks 48

F = fine-tune shape (N_seq=512, N_res=384), I = initial-training shape
(N_seq=128, N_res=256); c_m=256, c_z=128, 8 heads, OPM dim 32, bf16, one
recycle.  The step (fwd+bwd+Adam) is captured in a CUDA graph and replayed."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200.model import ModelConfig  # noqa: E402
from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer  # noqa: E402

SHAPES = {"I": (128, 256), "F": (512, 384)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="F", choices=sorted(SHAPES))
    ap.add_argument("--blocks", type=int, default=48)
    ap.add_argument("--recompute", action="store_true")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    S, R = SHAPES[args.shape]
    cfg = ModelConfig(n_blocks=args.blocks, n_seq=S, n_res=R, c_m=256, c_z=128, heads=8, opm_dim=32)
    plan = ExecutionPlan(act_dtype="bf16", fixed_recycles=1,
                         recompute=("evoformer",) if args.recompute else ())
    tr = Trainer.create(cfg, plan)
    tr.stage_features(0)                       # pinned host features for device_step's H2D
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    if args.no_graph:
        def step():
            return tr.device_step(1)
        for _ in range(2):
            step()
    else:
        tr.capture(n_cycles=1, warmup=2)

        def step():
            tr.graph.replay()
            return tr.graph_loss
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    print(json.dumps({"shape": args.shape, "n_seq": S, "n_res": R, "blocks": args.blocks,
                      "recompute": args.recompute, "ms_per_step": round(ms, 2),
                      "samples_per_s": round(1e3 / ms, 3), "loss": float(loss.item()),
                      "weights_etc_gb": round(base / 1e9, 2),
                      "peak_gb": round(torch.cuda.max_memory_allocated() / 1e9, 2),
                      "peak_reserved_gb": round(torch.cuda.max_memory_reserved() / 1e9, 2)}))


if __name__ == "__main__":
    main()
