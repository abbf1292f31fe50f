"""A/B the gradients of one bench-shape fwd+bwd (2 blocks) with an engine switch on/off:
    CMP_VAR=EVO_OPM_DNUM_TC python tools/cmp_stream.py     (default switch: EVO_GLUE_STREAM)"""
import os, sys, subprocess, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import torch
    from paper_2207_05477_b200.model import ModelConfig
    from paper_2207_05477_b200.trainer import ExecutionPlan, Trainer
    cfg = ModelConfig(n_blocks=2, n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32)
    tr = Trainer.create(cfg, ExecutionPlan(act_dtype="bf16", fixed_recycles=1))
    loss, _ = tr.engine.forward_backward(tr.feats, 1)
    torch.cuda.synchronize()
    np.save(sys.argv[1], tr.store.regions["grads"].cpu().numpy())
    print("loss", float(loss))
else:
    for e in ("1", "0"):
        subprocess.run([sys.executable, __file__, f"/tmp/g{e}.npy"], env=dict(os.environ, **{os.environ.get("CMP_VAR", "EVO_GLUE_STREAM"): e}), check=True)
    a, b = np.load("/tmp/g1.npy"), np.load("/tmp/g0.npy")
    from paper_2207_05477_b200.model import ModelConfig, flatten_params
    from paper_2207_05477_b200.fusion import build_layout
    cfg = ModelConfig(n_blocks=2, n_seq=128, n_res=256, c_m=256, c_z=128, heads=8, opm_dim=32)
    slots = build_layout(list(flatten_params(cfg)))
    worst = []
    for s in slots:
        lo = s.offset // 4; n = int(np.prod(s.shape)) if s.shape else 1
        x, y = a[lo:lo+n], b[lo:lo+n]
        d = np.abs(x - y).max() / max(np.abs(y).max(), 1e-30)
        worst.append((d, s.name))
    worst.sort(reverse=True)
    gmax = np.abs(b).max()
    print(f"global: max|diff| / max|g| = {np.abs(a - b).max() / gmax:.3e}  (gmax {gmax:.3e})")
    w2 = []
    for s_ in slots:
        lo = s_.offset // 4; n = int(np.prod(s_.shape)) if s_.shape else 1
        w2.append((np.abs(a[lo:lo+n] - b[lo:lo+n]).max() / max(np.abs(b[lo:lo+n]).max(), 1e-3 * gmax), s_.name))
    w2.sort(reverse=True)
    print("floored at 1e-3 gmax:", [(f"{d:.2e}", n) for d, n in w2[:6]])
    for d, n in worst[:12]: print(f"{d:.3e} {n}")
