"""Per-parameter error of the bf16 / f32 engine with TriangleMultiplication
against the oracle restatement (the test_block_with_trimul_matches_oracle
configuration), worst ten first.

    python tools/trimul_errs.py [bf16|f32] [seed]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle import evoformer_np as O  # noqa: E402
from paper_2207_05477_b200.model import ModelConfig  # noqa: E402
from conftest import rel_err  # noqa: E402
from test_gpu_parity import _run_engine  # noqa: E402


def main(dtype="bf16", seed=7, trimul=True):
    kw = dict(n_blocks=1, n_seq=32, n_res=64, c_m=64, c_z=32, heads=2, opm_dim=32, trimul=trimul)
    cfg, ocfg = ModelConfig(**kw), O.ModelConfig(**kw)
    oloss, ograds, (omsa, opair) = O.serial_grads(ocfg, O.init_params(ocfg, seed), O.make_features(ocfg, 3))
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    loss, msa, pair, grads = _run_engine(cfg, seed, 3, 1, dt)
    gmax = max(np.abs(v).max() for v in ograds.values())
    errs = {n: rel_err(grads[n], ograds[n], 1e-3 * gmax) for n in ograds}
    print(f"{dtype} trimul={trimul} seed={seed}: pair {rel_err(pair.reshape(opair.shape), opair):.2e} "
          f"msa {rel_err(msa.reshape(omsa.shape), omsa):.2e} median grad {np.median(list(errs.values())):.2e}")
    for n in sorted(errs, key=errs.get, reverse=True)[:10]:
        print(f"  {errs[n]:.3e}  {n}  max|g|={np.abs(ograds[n]).max():.3e}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "bf16", int(sys.argv[2]) if len(sys.argv) > 2 else 7,
         (sys.argv[3] != "0") if len(sys.argv) > 3 else True)
