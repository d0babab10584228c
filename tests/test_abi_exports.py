"""The C-ABI libraries load and export every symbol include/*.h declares
(CPU only: no compute calls)."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2211_10017_b200")

_DECL = re.compile(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(moe_\w+)\s*\(", re.M)


def declared(header):
    src = open(header).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//[^\n]*", "", src)
    return sorted(set(m.group(1) for m in _DECL.finditer(src)) - {"moe_layer_desc"})


HEADERS = {os.path.join(ROOT, "include", "moe_cuda.h"): os.path.join(PKG, "libmoe_cuda.so")}
if os.path.exists(os.path.join(ROOT, "include", "moe_ep.h")):
    HEADERS[os.path.join(ROOT, "include", "moe_ep.h")] = os.path.join(PKG, "libmoe_ep.so")


@pytest.mark.parametrize("header", sorted(HEADERS))
def test_library_exports_every_declared_symbol(header):
    lib_path = HEADERS[header]
    assert os.path.exists(lib_path), f"{lib_path} not built (make / __graft_entry__.build())"
    lib = ctypes.CDLL(lib_path)
    names = declared(header)
    assert len(names) > 5
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_abi_table_matches_header():
    from paper_2211_10017_b200 import abi
    names = set(declared(os.path.join(ROOT, "include", "moe_cuda.h")))
    assert names == set(abi._SIGS), names ^ set(abi._SIGS)


def test_no_device_is_an_error_not_a_fallback():
    """Without a GPU the library reports a CUDA error instead of computing."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2211_10017_b200 import abi
    sm = ctypes.c_int()
    st = abi.lib().moe_cuda_device_info(ctypes.byref(sm), None, None)
    assert st == abi.MOE_ECUDA
    assert "CUDA" in abi.last_error()


def test_missing_extension_fails_loudly(tmp_path, monkeypatch):
    from paper_2211_10017_b200 import abi
    monkeypatch.setattr(abi, "_lib", None)
    monkeypatch.setattr(abi, "LIB_PATH", str(tmp_path / "libmoe_cuda.so"))
    with pytest.raises(ImportError):
        abi.lib()


def test_headers_have_no_torch_types():
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        assert "torch" not in src.lower().replace("no torch types", "")
        assert "at::" not in src and "Tensor" not in src
