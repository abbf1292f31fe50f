"""Per-tensor errors of one Evoformer block at the bench shape (I) against the
CPU oracle, sorted (diagnostic for tests/test_gpu_bench_shape.py).

    python tools/parity_I.py [f32|bf16]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import grad_err, rel_err  # noqa: E402
from test_gpu_bench_shape import SHAPE_I, _engine_I  # noqa: E402
from oracle import evoformer_np as O  # noqa: E402


def main():
    dt = torch.float32 if (sys.argv[1:] or ["f32"])[0] == "f32" else torch.bfloat16
    ocfg = O.ModelConfig(**SHAPE_I)
    oloss, ograds, (omsa, opair) = O.serial_grads(ocfg, O.init_params(ocfg, 7), O.make_features(ocfg, 3))
    loss, msa, pair, grads = _engine_I(dt)
    G = max(float(np.abs(g).max()) for g in ograds.values())
    print("msa", rel_err(msa.reshape(omsa.shape), omsa), "pair", rel_err(pair.reshape(opair.shape), opair),
          "loss", abs(loss - oloss) / abs(oloss))
    errs = {n: grad_err(grads[n].reshape(g.shape), g, n, 1e-6, G) for n, g in ograds.items()}
    for n in sorted(errs, key=errs.get)[-20:]:
        print(f"{errs[n]:.3e}  {n}  max|ref|={np.abs(ograds[n]).max():.3e}")


if __name__ == "__main__":
    main()
