"""Per-kernel breakdown of the TriangleMultiplication workload (4 blocks with
trimul on minus the same without): python tools/step_profile_trimul.py"""
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200.model import ModelConfig  # noqa: E402
from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer  # noqa: E402


def prof(trimul):
    cfg = ModelConfig(n_blocks=4, n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32, trimul=trimul)
    tr = Trainer.create(cfg, ExecutionPlan(act_dtype="bf16", fixed_recycles=1))
    for _ in range(2):
        tr.engine.forward_backward(tr.feats, 1)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as p:
        tr.engine.forward_backward(tr.feats, 1)
        torch.cuda.synchronize()
    agg = defaultdict(lambda: [0, 0.0])
    for e in p.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            n = e.name.replace("void ", "").replace("(anonymous namespace)::", "").replace("evo::", "").split("(")[0][:80]
            agg[n][0] += 1
            agg[n][1] += e.device_time_total
    return agg


a, b = prof(True), prof(False)
rows = []
for k in a:
    dn = a[k][0] - b.get(k, [0, 0])[0]
    dt = a[k][1] - b.get(k, [0, 0.0])[1]
    if dn > 0 or dt > 20:
        rows.append((dt, dn, k))
tot = sum(r[0] for r in rows)
print(f"TriMul extra kernel time, 4 blocks: {tot / 1e3:.3f} ms")
for dt, dn, k in sorted(rows, reverse=True):
    print(f"{dt / 1e3:8.3f} ms  +{dn:4d}  {k}")
