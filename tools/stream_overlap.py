"""Kernel timeline of one training step (n blocks): per-stream busy time,
union busy time, overlap and idle gaps.
    python tools/stream_overlap.py [n_blocks]"""
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200.model import ModelConfig  # noqa: E402
from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer  # noqa: E402


def main(n_blocks=4):
    cfg = ModelConfig(n_blocks=int(n_blocks), n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32)
    tr = Trainer.create(cfg, ExecutionPlan(act_dtype="bf16", fixed_recycles=1))
    for _ in range(2):
        tr.engine.forward_backward(tr.feats, 1)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        tr.engine.forward_backward(tr.feats, 1)
        torch.cuda.synchronize()
    ev = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0:
            ev.append((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0) or 0))
    ev.sort()
    t0, t1 = ev[0][0], max(e[1] for e in ev)
    per = defaultdict(float)
    for a, b, sid in ev:
        per[sid] += b - a
    # union of intervals
    union, cur_a, cur_b = 0.0, None, None
    for a, b, _ in ev:
        if cur_b is None or a > cur_b:
            if cur_b is not None:
                union += cur_b - cur_a
            cur_a, cur_b = a, b
        else:
            cur_b = max(cur_b, b)
    union += cur_b - cur_a
    span = t1 - t0
    print(f"span {span / 1e3:.2f} ms, union busy {union / 1e3:.2f} ms ({100 * union / span:.1f}%), "
          f"sum kernel time {sum(per.values()) / 1e3:.2f} ms")
    for sid, t in sorted(per.items(), key=lambda x: -x[1]):
        print(f"  stream {sid}: {t / 1e3:.2f} ms")
    print(f"overlap (sum - union) {(sum(per.values()) - union) / 1e3:.2f} ms; idle {(span - union) / 1e3:.2f} ms")


if __name__ == "__main__":
    main(*sys.argv[1:])
