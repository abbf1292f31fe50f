"""CPU checks of the reference block-module API surface
(``paper_2207_05477_b200.modules``, src/model.py:140-259): parameter
dataclasses, flatten order, bit-identical init, branch ownership, the serial
adapter and the activation-dtype context.  The compute paths are covered on
the GPU by tests/test_gpu_modules.py."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _cfg(**kw):
    from paper_2207_05477_b200.model import ModelConfig
    base = dict(n_blocks=2, n_seq=8, n_res=16, c_m=32, c_z=16, heads=4, opm_dim=4)
    base.update(kw)
    return ModelConfig(**base)


def test_flatten_params_order_and_init_bit_identical():
    from paper_2207_05477_b200 import modules as Mo
    from paper_2207_05477_b200.model import flatten_params, init_params
    cfg = _cfg()
    mp = Mo.init_params(cfg, 7, device="cpu")
    flat = init_params(cfg, 7)
    named = Mo.flatten_params(mp)
    assert [n for n, _ in named] == [n for n, _ in flatten_params(cfg)]
    for n, t in named:
        assert t.dtype == torch.float32 and t.requires_grad
        assert np.array_equal(t.detach().numpy(), flat[n]), n
    msa, pair = Mo.branch_param_names(mp, "msa"), Mo.branch_param_names(mp, "pair")
    assert not (msa & pair) and msa | pair == {n for n, _ in named}


def test_flatten_params_matches_reference_names():
    """Same (name, shape) list as the reference's flatten_params."""
    import os
    import sys
    src = "/root/reference/pkg/src"
    if os.path.isdir(src) and src not in sys.path:
        sys.path.append(src)
    ref = pytest.importorskip("evotrain.model", reason="reference package not importable here")
    from paper_2207_05477_b200 import modules as Mo
    kw = dict(n_blocks=2, n_seq=8, n_res=16, c_m=32, c_z=16, heads=4, opm_dim=4)
    rmp = ref.init_params(ref.ModelConfig(**kw), 7)
    mp = Mo.init_params(_cfg(**kw), 7, device="cpu")
    got = [(n, tuple(t.shape)) for n, t in Mo.flatten_params(mp)]
    want = [(n, tuple(t.shape)) for n, t in ref.flatten_params(rmp)]
    assert got == want
    for (n, t), (_, rt) in zip(Mo.flatten_params(mp), ref.flatten_params(rmp)):
        assert np.array_equal(t.detach().numpy(), rt.data), n


def test_trimul_params_are_pair_branch():
    from paper_2207_05477_b200 import modules as Mo
    mp = Mo.init_params(_cfg(trimul=True), 7, device="cpu")
    names = [n for n, _ in Mo.flatten_params(mp)]
    tm = [n for n in names if ".tri_mul_" in n]
    assert len(tm) == 2 * 2 * 16
    assert set(tm) <= Mo.branch_param_names(mp, "pair")


def test_serial_adapter_and_dtype_context():
    from paper_2207_05477_b200 import modules as Mo
    from paper_2207_05477_b200.errors import ContractError
    par = Mo.SerialPar()
    x = object()
    assert par.allgather(x, 1, "m") is x and par.reducescatter_sum(x, 1, "m") is x
    assert par.alltoall(x, 2, 1, "m") is x and par.slice_np(x, 1) is x
    assert Mo.act_dtype() == torch.float32
    with Mo.activation_dtype(torch.bfloat16):
        assert Mo.act_dtype() == torch.bfloat16
    assert Mo.act_dtype() == torch.float32
    with pytest.raises(ContractError):
        Mo.set_act_dtype(torch.float16)

    class Sharded:
        size, index = 2, 0
    with pytest.raises(ContractError):
        Mo._serial(Sharded())
