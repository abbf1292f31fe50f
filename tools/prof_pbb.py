"""Drive the pair-bias backward stream kernel once per layout at the bench
pair shape (R=256, c_z=128, H=8; dz16 and the column sums emitted as on the
engine path), for ncu captures:

    ncu --set full --import-source on -k regex:pair_bias_bwd -o pbb python tools/prof_pbb.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import ops  # noqa: E402


def main():
    R, cz, H, dev = 256, 128, 8, "cuda"
    z = torch.randn(R * R, cz, device=dev).to(torch.bfloat16)
    g, b = torch.ones(cz, device=dev), torch.zeros(cz, device=dev)
    w = torch.randn(cz, H, device=dev) * 0.1
    nb, mean, rstd = ops.pair_bias_fwd(z, g, b, w, R, H, False)
    dnb = torch.randn(H, R, R, device=dev)
    dz = torch.randn(R * R, cz, device=dev)
    dw = torch.empty(cz, H, device=dev)
    dz16 = torch.empty(R * R, cz, device=dev, dtype=torch.bfloat16)
    dzsum = torch.empty(cz, device=dev)
    for swap in (False, True):
        ops.pair_bias_bwd(z, mean, rstd, g, b, w, dnb, swap, dz, g.clone(), b.clone(), dw, R, H,
                          dz16=dz16, dzsum=dzsum)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
