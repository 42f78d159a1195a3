"""B200-native MoE-layer inference path (arXiv 2303.06182, dynamic gating).

C-ABI boundary: include/moe_capi.h (``libmoe_b200.so``, sm_100a kernels).
C++ drop-in of the reference API: include/moesim/gating.hpp
(``libmoesim_b200.so``).  Python host mirror: ``gating`` (reference function
names) and ``layer.MoeLayer`` (device-resident perf path).
"""
from ._capi import MoeError, MoeInvalidArgument, load  # noqa: F401

__all__ = ["MoeError", "MoeInvalidArgument", "load"]
