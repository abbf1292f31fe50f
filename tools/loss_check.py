"""Per-step training loss of the bench workload (fewer blocks optional):
    python tools/loss_check.py [n_blocks] [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200.model import ModelConfig  # noqa: E402
from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer  # noqa: E402


def main(n_blocks=48, steps=4):
    cfg = ModelConfig(n_blocks=int(n_blocks), n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32)
    tr = Trainer.create(cfg, ExecutionPlan(act_dtype="bf16", fixed_recycles=1))
    for k in range(int(steps)):
        loss, (msa, pair) = tr.engine.forward_backward(tr.feats, 1)
        g = tr.store.regions["grads"]
        print(k, float(loss), "msa finite", bool(torch.isfinite(msa.float()).all()), "pair finite",
              bool(torch.isfinite(pair.float()).all()), "grad finite", bool(torch.isfinite(g).all()),
              "gmax", float(g.abs().max()))
        tr.store.step()


if __name__ == "__main__":
    main(*sys.argv[1:])
