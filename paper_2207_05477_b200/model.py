"""Model configuration, parameter naming/initialisation and synthetic
features -- the reference's ``evotrain.model`` surface (src/model.py).

Parameters are identified by the reference's flatten names
(``block{i}.{module}.{field}`` / ``...attn.{wq,...}``, src/model.py:203-220)
and initialised with the same splitmix64 draws (src/model.py:140-200), so
the GPU model starts from bit-identical weights and features.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ContractError
from .prng import Prng, splitmix64

MSA_BRANCH_MODULES = ("row_attn", "col_attn", "msa_trans", "opm")
PAIR_BRANCH_MODULES = ("tri_start", "tri_end", "pair_trans")
TRIMUL_MODULES = ("tri_mul_out", "tri_mul_in")
ATTN_FIELDS = ("wq", "wk", "wv", "wg", "bg", "wo", "bo")
_TRIMUL_SEED_SALT = 0x5EED7A1


@dataclass
class ModelConfig:
    """src/model.py:42-65.  ``trimul`` is the extension switch for
    TriangleMultiplication (absent from the reference; default off)."""

    n_blocks: int = 2
    n_seq: int = 8
    n_res: int = 8
    c_m: int = 8
    c_z: int = 8
    heads: int = 2
    opm_dim: int = 4
    transition_factor: int = 4
    feat_dim: int = 8
    pad_fraction: float = 0.1
    trimul: bool = False
    trimul_hidden: int = 0

    @property
    def head_dim_m(self) -> int:
        return self.c_m // self.heads

    @property
    def head_dim_z(self) -> int:
        return self.c_z // self.heads

    @property
    def c_hidden_mul(self) -> int:
        return self.trimul_hidden or self.c_z

    def validate(self):
        if self.c_m % self.heads or self.c_z % self.heads:
            raise ContractError("channel dims must be divisible by heads")


@dataclass
class ExecPolicy:
    """src/model.py:68-73.  ``fused`` is accepted for API parity; the GPU
    path is always the fused operator (one kernel family per module)."""

    fused: bool = True
    row_chunk: int = 0


def param_specs(cfg: ModelConfig):
    """[(name, shape, init)] in the reference flatten order (src/model.py:203-220);
    init is 'u' (uniform*0.1, reference draw order), 'tu' (TriMul extension
    stream), 'ones' or 'zeros'."""
    H = cfg.heads
    specs = [
        ("msa_embed.w", (cfg.feat_dim, cfg.c_m), "u"), ("msa_embed.b", (cfg.c_m,), "zeros"),
        ("pair_embed.w", (cfg.feat_dim, cfg.c_z), "u"), ("pair_embed.b", (cfg.c_z,), "zeros"),
        ("recycle_m.g", (cfg.c_m,), "ones"), ("recycle_m.b", (cfg.c_m,), "zeros"),
        ("recycle_z.g", (cfg.c_z,), "ones"), ("recycle_z.b", (cfg.c_z,), "zeros"),
    ]

    def attn(prefix, c, bias_from):
        hd = c // H
        out = [(f"{prefix}.ln_g", (c,), "ones"), (f"{prefix}.ln_b", (c,), "zeros")]
        out += [(f"{prefix}.attn.{f}", (c, H, hd), "u") for f in ("wq", "wk", "wv", "wg")]
        out += [(f"{prefix}.attn.bg", (H, hd), "zeros"), (f"{prefix}.attn.wo", (H, hd, c), "u"),
                (f"{prefix}.attn.bo", (c,), "zeros")]
        if bias_from:
            out += [(f"{prefix}.bias_ln_g", (bias_from,), "ones"),
                    (f"{prefix}.bias_ln_b", (bias_from,), "zeros"),
                    (f"{prefix}.w_bias", (bias_from, H), "u")]
        return out

    def trans(prefix, c):
        f = cfg.transition_factor
        return [(f"{prefix}.ln_g", (c,), "ones"), (f"{prefix}.ln_b", (c,), "zeros"),
                (f"{prefix}.w1", (c, f * c), "u"), (f"{prefix}.b1", (f * c,), "zeros"),
                (f"{prefix}.w2", (f * c, c), "u"), (f"{prefix}.b2", (c,), "zeros")]

    def trimul(prefix, cz, ch):
        out = [(f"{prefix}.ln_in_g", (cz,), "ones"), (f"{prefix}.ln_in_b", (cz,), "zeros")]
        for nm in ("ap", "ag", "bp", "bg"):
            out += [(f"{prefix}.w_{nm}", (cz, ch), "tu"), (f"{prefix}.b_{nm}", (ch,), "zeros")]
        out += [(f"{prefix}.ln_out_g", (ch,), "ones"), (f"{prefix}.ln_out_b", (ch,), "zeros"),
                (f"{prefix}.w_o", (ch, cz), "tu"), (f"{prefix}.b_o", (cz,), "zeros"),
                (f"{prefix}.w_g", (cz, cz), "tu"), (f"{prefix}.b_g", (cz,), "zeros")]
        return out

    k = cfg.opm_dim
    for i in range(cfg.n_blocks):
        p = f"block{i}"
        specs += attn(f"{p}.row_attn", cfg.c_m, cfg.c_z)
        specs += attn(f"{p}.col_attn", cfg.c_m, 0)
        specs += trans(f"{p}.msa_trans", cfg.c_m)
        specs += [(f"{p}.opm.ln_g", (cfg.c_m,), "ones"), (f"{p}.opm.ln_b", (cfg.c_m,), "zeros"),
                  (f"{p}.opm.w_left", (cfg.c_m, k), "u"), (f"{p}.opm.b_left", (k,), "zeros"),
                  (f"{p}.opm.w_right", (cfg.c_m, k), "u"), (f"{p}.opm.b_right", (k,), "zeros"),
                  (f"{p}.opm.w_out", (k * k, cfg.c_z), "u"), (f"{p}.opm.b_out", (cfg.c_z,), "zeros")]
        specs += attn(f"{p}.tri_start", cfg.c_z, cfg.c_z)
        specs += attn(f"{p}.tri_end", cfg.c_z, cfg.c_z)
        specs += trans(f"{p}.pair_trans", cfg.c_z)
        if cfg.trimul:
            for m in TRIMUL_MODULES:
                specs += trimul(f"{p}.{m}", cfg.c_z, cfg.c_hidden_mul)
    return specs


def init_params(cfg: ModelConfig, seed: int) -> dict:
    """src/model.py:172-200 -> {name: float32 ndarray} in flatten order."""
    cfg.validate()
    rng = Prng(seed)
    trng = Prng(seed ^ _TRIMUL_SEED_SALT)
    out = {}
    for name, shape, kind in param_specs(cfg):
        if kind == "u":
            out[name] = rng.uniform(shape) * np.float32(0.1)
        elif kind == "tu":
            out[name] = trng.uniform(shape) * np.float32(0.1)
        elif kind == "ones":
            out[name] = np.ones(shape, np.float32)
        else:
            out[name] = np.zeros(shape, np.float32)
    return out


def flatten_params(cfg: ModelConfig) -> list:
    """[(name, shape)] in the reference flatten order (src/model.py:203-220)."""
    return [(n, s) for n, s, _ in param_specs(cfg)]


def branch_param_names(cfg: ModelConfig, branch: str) -> set:
    """src/model.py:223-236 (TriMul, when enabled, belongs to the pair branch)."""
    embeds = {"msa": ("msa_embed.", "recycle_m."), "pair": ("pair_embed.", "recycle_z.")}[branch]
    mods = MSA_BRANCH_MODULES if branch == "msa" else PAIR_BRANCH_MODULES + TRIMUL_MODULES
    names = set()
    for name, _, _ in param_specs(cfg):
        if name.startswith(embeds) or (name.startswith("block") and name.split(".")[1] in mods):
            names.add(name)
    return names


@dataclass
class Features:
    msa_feat: np.ndarray  # [1, S, R, F]
    pair_feat: np.ndarray  # [1, R, R, F]
    msa_mask: np.ndarray  # [1, S, R]
    pair_mask: np.ndarray  # [1, R, R]


def make_features(cfg: ModelConfig, seed: int) -> Features:
    """src/model.py:274-288."""
    rng = Prng(seed)
    s, r, f = cfg.n_seq, cfg.n_res, cfg.feat_dim
    n_valid = r - int(np.floor(cfg.pad_fraction * r))
    msa_mask = np.ones((1, s, r), np.float32)
    msa_mask[:, :, n_valid:] = 0.0
    pair_mask = np.ones((1, r, r), np.float32)
    pair_mask[:, n_valid:, :] = 0.0
    pair_mask[:, :, n_valid:] = 0.0
    msa_feat = rng.uniform((1, s, r, f))
    pair_feat = rng.uniform((1, r, r, f))
    return Features(msa_feat, pair_feat, msa_mask, pair_mask)


def draw_num_recycles(base_seed: int, step: int) -> int:
    """src/model.py:291-293."""
    return 1 + int(splitmix64(base_seed + step, 1)[0] % 4)


def step_feature_seed(base_seed: int, step: int) -> int:
    """src/trainer.py:98-101."""
    return int(splitmix64(base_seed + step, 2)[1] & 0x7FFFFFFF)
