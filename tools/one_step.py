"""One bench-shape training step on n blocks (for ncu captures of the glue kernels).

    python tools/one_step.py [n_blocks]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200.model import ModelConfig  # noqa: E402
from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer  # noqa: E402


def main(n_blocks=1):
    cfg = ModelConfig(n_blocks=int(n_blocks), n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32)
    tr = Trainer.create(cfg, ExecutionPlan(act_dtype="bf16", fixed_recycles=1))
    tr.engine.forward_backward(tr.feats, 1)
    tr.store.step()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(*sys.argv[1:])
