"""B200-native discrete X-ray transform (arXiv 2006.00686): forward, adjoint, CSR dump.

Product path: ``Plan`` (plan.py) -> ctypes -> libxrt.so (csrc/, sm_100a CUDA).
Multi-GPU view sharding: ``dist.ShardedPlan`` (torch.distributed / NCCL).
This package never imports ``oracle/`` and has no CPU fallback.
"""
from .plan import Plan, version  # noqa: F401
from ._lib import XrtError  # noqa: F401
