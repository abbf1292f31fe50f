"""smoke() configuration with the per-parameter gradient errors listed."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import evoformer_np as O  # noqa: E402
from paper_2207_05477_b200.engine import BlockEngine, DeviceFeatures  # noqa: E402
from paper_2207_05477_b200.fusion import FusionEngine  # noqa: E402
from paper_2207_05477_b200.model import ModelConfig, flatten_params, init_params, make_features  # noqa: E402

cfg = ModelConfig(n_blocks=1, n_seq=16, n_res=32, c_m=64, c_z=32, heads=2, opm_dim=8)
P = init_params(cfg, 7)
feats = make_features(cfg, 3)
st = FusionEngine([(n, P[n]) for n, _ in flatten_params(cfg)], shadow_dtype=torch.float32)
eng = BlockEngine(cfg, st, torch.float32)
loss, (msa, pair) = eng.forward_backward(DeviceFeatures(feats, "cuda", cfg), 1)
torch.cuda.synchronize()
ocfg = O.ModelConfig(n_blocks=1, n_seq=16, n_res=32, c_m=64, c_z=32, heads=2, opm_dim=8)
oloss, ograds, _ = O.serial_grads(ocfg, O.init_params(ocfg, 7), O.make_features(ocfg, 3))
gmax = max(np.abs(v).max() for v in ograds.values())
errs = []
for n in ograds:
    a, b = st.grad(n).cpu().numpy().astype(np.float64), np.asarray(ograds[n], np.float64)
    e = float(np.abs(a - b).max() / max(np.abs(a).max(), np.abs(b).max(), 1e-6 * gmax, 1e-30))
    errs.append((e, n, float(np.abs(b).max())))
for e in sorted(errs, reverse=True)[:8]:
    print(f"{e[0]:.3e} {e[1]} max|g|={e[2]:.3e} gmax={gmax:.3e}")
