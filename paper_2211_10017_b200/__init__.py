"""B200-native (sm_100a) MoE-layer inference hot path of arXiv 2211.10017.

* ``ops`` / ``MoELayer``  -- device-resident path over the C-ABI
  (include/moe_cuda.h, libmoe_cuda.so);
* ``_moeinfer``            -- drop-in for the reference's pybind module
  (same names as proj/bindings/py_module.cpp), built by ``make``.
"""
from . import abi  # noqa: F401

__all__ = ["abi"]
