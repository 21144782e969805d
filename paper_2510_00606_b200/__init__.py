"""elaskit-b200: B200-native per-step data-parallel recovery path of ElasWave
(arXiv 2510.00606) behind the reference's elaskit API.

Layout
  include/elaskit/*.hpp, include/ew_api.h   C++ API (drop-in) and C ABI
  paper_2510_00606_b200/csrc/               C++ planners + sm_100a kernels
  paper_2510_00606_b200/libelaskit_b200.so  the built library (in-tree)
  fabric.py / device.py / reshard.py        Python view of the same API
"""
from . import _native  # noqa: F401  (fails loudly when the library is missing)
from .fabric import (CommGroup, PartitionLayout, SnapshotRing, TransferPlan,  # noqa: F401
                     contiguous_layout, draw, integrity_check, interleaved_layout,
                     overlap_matrix, philox4x64, plan_edit, reshard_copies,
                     reshard_microbatches, weighted_grad_average)

LIB_PATH = str(_native.LIB_PATH)
__version__ = "0.1.0"
