"""CPU-side checks of the C-ABI library: it loads without a GPU and exports
every symbol include/evoformer_sm100.h declares, all bound in _lib.SIGNATURES."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "evoformer_sm100.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(evo_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2207_05477_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2207_05477_b200 import build
        build.build(verbose=False)
    return _lib.load()


def test_header_declares_the_path():
    names = declared_functions()
    for must in ("evo_attn_fwd", "evo_attn_bwd", "evo_layernorm_fwd", "evo_gemm",
                 "evo_adam_clip_ema", "evo_sumsq_f64", "evo_opm_norm_fwd", "evo_pair_bias_fwd"):
        assert must in names


def test_every_declared_symbol_is_exported_and_bound(lib):
    from paper_2207_05477_b200 import _lib
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from _lib.SIGNATURES"


def test_bound_signatures_exist_in_header():
    from paper_2207_05477_b200 import _lib
    declared = set(declared_functions())
    assert set(_lib.SIGNATURES) <= declared


def test_host_only_queries(lib):
    assert lib.evo_version() >= 1
    assert lib.evo_layernorm_bwd_workspace(100, 256) >= 256 * 2 * 256 * 4
    assert lib.evo_attn_bwd_workspace(4, 64, 2, 32, 1) > 0


def test_device_check_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2207_05477_b200 import _lib
    from paper_2207_05477_b200.errors import NativeUnavailable
    _lib._device_ok = None
    with pytest.raises(NativeUnavailable):
        _lib.lib()
