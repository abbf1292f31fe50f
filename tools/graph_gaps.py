"""Idle time between kernels inside the CUDA-graph-replayed training step
(the bench's timed path): span, union of kernel intervals, idle gaps.

    python tools/graph_gaps.py [n_blocks]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200.model import ModelConfig  # noqa: E402
from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer  # noqa: E402


def main(n_blocks=8):
    cfg = ModelConfig(n_blocks=int(n_blocks), n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32)
    tr = Trainer.create(cfg, ExecutionPlan(act_dtype="bf16", fixed_recycles=1))
    tr.capture(n_cycles=1, warmup=2)
    for _ in range(3):
        tr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tr.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"graph replay (no profiler): {e0.elapsed_time(e1):.3f} ms")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        tr.replay()
        torch.cuda.synchronize()
    ev = sorted((e.time_range.start, e.time_range.end) for e in prof.events()
                if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0)
    span = max(b for _, b in ev) - ev[0][0]
    union, ca, cb = 0.0, None, None
    gaps = []
    for a, b in ev:
        if cb is None or a > cb:
            if cb is not None:
                union += cb - ca
                gaps.append(a - cb)
            ca, cb = a, b
        else:
            cb = max(cb, b)
    union += cb - ca
    gaps.sort(reverse=True)
    print(f"kernels {len(ev)}, span {span / 1e3:.3f} ms, union busy {union / 1e3:.3f} ms, idle {(span - union) / 1e3:.3f} ms "
          f"in {len(gaps)} gaps (largest {[round(g, 1) for g in gaps[:8]]} us, median {gaps[len(gaps) // 2]:.2f} us)")


if __name__ == "__main__":
    main(*sys.argv[1:])
