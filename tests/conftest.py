import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# deterministic algorithm choice for any library GEMM path in every (spawned)
# test process: no timing-dependent selection (inherited by mp.spawn workers)
os.environ.setdefault("EVO_GEMM_TUNE", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def rel_err(a, b, floor=0.0):
    """max|a-b| / max(max|a|, max|b|, floor) -- the reference's inf-norm metric
    (tests/test_acceptance.py:67-69) with the survey's denominator floor."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    denom = max(np.abs(a).max(initial=0.0), np.abs(b).max(initial=0.0), floor, 1e-30)
    return float(np.abs(a - b).max(initial=0.0) / denom)


@pytest.fixture
def golden():
    return load_golden


# gradients that are analytically zero: bias_ln_b of every pair-bias module is
# a per-head constant shift of the logits, which softmax ignores (SURVEY.md
# section 0.5); both sides hold rounding noise, so they are measured against G
ANALYTIC_ZERO = ("bias_ln_b",)


def grad_err(a, b, name, floor_frac, G):
    if any(name.endswith(z) for z in ANALYTIC_ZERO):
        return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max(initial=0.0) / max(G, 1e-30))
    return rel_err(a, b, floor_frac * G)


def slot_errs(store, flat, ref, floor_frac):
    """Per-parameter floored errors of a flat pooled grad region against
    ``ref`` (another flat region with the same layout, or a name -> array dict
    such as the oracle's grads): err(t) = max|a-b| / max(max|a|, max|b|,
    floor_frac * G), G = max|ref| over all parameters.
    A wrong, missing or double-counted small-magnitude slot cannot hide behind
    the largest gradient of the region."""
    flat = np.asarray(flat)
    views = {}
    for s in store.slots:
        n = int(np.prod(s.shape, dtype=np.int64)) if s.shape else 1
        lo = s.offset // 4
        views[s.name] = (lo, n, s.shape)
    if isinstance(ref, dict):
        refs = {k: np.asarray(ref[k]).ravel() for k in views}
    else:
        refs = {k: np.asarray(ref)[lo:lo + n] for k, (lo, n, _) in views.items()}
    G = max(float(np.abs(r).max(initial=0.0)) for r in refs.values())
    return {k: grad_err(flat[lo:lo + n], refs[k], k, floor_frac, G) for k, (lo, n, _) in views.items()}
