"""Print per-parameter relative errors of the GPU engine vs a golden file."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import load_golden, rel_err  # noqa: E402
from paper_2207_05477_b200.engine import BlockEngine, DeviceFeatures  # noqa: E402
from paper_2207_05477_b200.fusion import FusionEngine  # noqa: E402
from paper_2207_05477_b200.model import (ModelConfig, flatten_params, init_params,  # noqa: E402
                                         make_features)


def main(fname="model_O.npz", dtype="f32", top=25):
    top = int(top)
    g = load_golden(fname)
    nb, s, r, cm, cz, h, k, ncyc, fseed, pseed = (int(v) for v in g["cfg"])
    cfg = ModelConfig(n_blocks=nb, n_seq=s, n_res=r, c_m=cm, c_z=cz, heads=h, opm_dim=k)
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    P = init_params(cfg, pseed)
    st = FusionEngine([(n, P[n]) for n, _ in flatten_params(cfg)], shadow_dtype=dt)
    eng = BlockEngine(cfg, st, dt)
    feats = DeviceFeatures(make_features(cfg, fseed), "cuda", cfg)
    loss, (msa, pair) = eng.forward_backward(feats, ncyc)
    torch.cuda.synchronize()
    print(fname, dtype, "loss", loss.item(), float(g["loss"]))
    print("msa", rel_err(msa.float().cpu().numpy().reshape(g["msa"].shape), g["msa"]),
          "pair", rel_err(pair.float().cpu().numpy().reshape(g["pair"].shape), g["pair"]))
    gmax = max(np.abs(g[f"g::{n}"]).max() for n, _ in flatten_params(cfg))
    errs = []
    for n, _ in flatten_params(cfg):
        a = st.grad(n).cpu().numpy()
        errs.append((rel_err(a, g[f"g::{n}"], 1e-6 * gmax), n, float(np.abs(a).max()),
                     float(np.abs(g[f"g::{n}"]).max())))
    for e in sorted(errs, reverse=True)[:top]:
        print(f"{e[0]:.3e}  {e[1]:40s} gpu_max={e[2]:.3e} ref_max={e[3]:.3e}")


if __name__ == "__main__":
    main(*sys.argv[1:])
