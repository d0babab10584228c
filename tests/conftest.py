"""Shared fixtures.  `-m gpu` tests need a B200 and the built libmoe_cuda.so;
`-m "not gpu"` tests run on CPU (oracle, golden fixtures, ABI exports,
gloo multi-process EP host logic)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref/libmoeref.so not built (reference sources absent)")
    return Reference()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_10017_b200 import abi
    abi.lib()  # raises if the extension is missing: no silent fallback
    return torch.device("cuda:0")


def bits16(a):
    return np.ascontiguousarray(a).view(np.uint16)


def to_np(t):
    """torch CUDA tensor -> numpy (float16 stays float16)."""
    import torch
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.float16:
        return t.view(torch.int16).numpy().view(np.float16)
    if t.dtype == torch.int32:
        return t.numpy().view(np.uint32)
    return t.numpy()


def to_dev(a, device="cuda"):
    import torch
    a = np.ascontiguousarray(a)
    if a.dtype == np.float16:
        return torch.from_numpy(a.view(np.int16)).to(device).view(torch.float16)
    if a.dtype == np.uint32:
        return torch.from_numpy(a.view(np.int32)).to(device)
    return torch.from_numpy(a).to(device)


def norm_err(got, want):
    """max|got - want| / max|want| in f64 (SURVEY.md §8d parity metric)."""
    g = np.asarray(got, np.float64)
    w = np.asarray(want, np.float64)
    den = max(np.abs(w).max(), 1e-30)
    return float(np.abs(g - w).max() / den)


def layer_err(got, want, x):
    """Normalized error of a MoE layer output, net of the final fp16 rounding:
    max(|got - want| - ulp16(want), 0) / max|want - x|.  Both sides round
    x + contribution to fp16 once, so a 1-ulp disagreement is rounding noise
    that the 1e-2 budget of the contribution must not be charged with (it
    dominates when the contribution is small, e.g. T=2)."""
    g = np.asarray(got, np.float64)
    w = np.asarray(want, np.float64)
    xf = np.asarray(x, np.float64)
    ulp = np.spacing(np.abs(np.asarray(want, np.float16))).astype(np.float64)
    excess = np.maximum(np.abs(g - w) - ulp, 0.0)
    den = max(np.abs(w - xf).max(), 1e-30)
    return float(excess.max() / den)
