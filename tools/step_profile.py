"""Per-kernel time breakdown of one training step (torch.profiler / CUPTI).

    python tools/step_profile.py [n_blocks] [out.txt]
"""
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200.model import ModelConfig  # noqa: E402
from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer  # noqa: E402


def main(n_blocks=4, out=None):
    n_blocks = int(n_blocks)
    cfg = ModelConfig(n_blocks=n_blocks, n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32)
    tr = Trainer.create(cfg, ExecutionPlan(act_dtype="bf16", fixed_recycles=1))
    for _ in range(2):
        tr.engine.forward_backward(tr.feats, 1)
        tr.store.step()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        tr.engine.forward_backward(tr.feats, 1)
        tr.store.step()
        torch.cuda.synchronize()
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            name = e.name
            for pre in ("void ", "(anonymous namespace)::", "evo::"):
                name = name.replace(pre, "")
            name = name.split("(")[0][:90]
            agg[name][0] += 1
            agg[name][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
            total += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    lines = [f"total kernel time {total/1e3:.2f} ms for {n_blocks} blocks (+optimizer)"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{t/1e3:9.3f} ms {100*t/total:6.2f}%  x{n:5d}  {name}")
    text = "\n".join(lines)
    print(text)
    if out:
        with open(out, "w") as fh:
            fh.write(text + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
