"""B200-native AMYTISS engine: MDP construction + finite-horizon Bellman synthesis
on sm_100a, behind the C ABI in include/gridmdp_b200.h (libgridmdp_b200.so).

``paper_2005_06191_b200.gridmdp`` mirrors the reference's C++ API for the hot
path; ``paper_2005_06191_b200.sharded`` runs it across GPUs (one process per
GPU, torch.distributed/NCCL all-gather of V per Bellman step).
"""
from . import gridmdp  # noqa: F401
from ._capi import LIB_PATH, CLI_PATH  # noqa: F401

__all__ = ["gridmdp", "LIB_PATH", "CLI_PATH"]
