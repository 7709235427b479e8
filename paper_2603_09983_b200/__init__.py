"""B200-native MoE-SpAc verification-step hot path.

Native pieces (built in-tree into ``_lib/libmoespac.so`` by ``build.py``):
  csrc/kernels/router_hist.cu   K1 router top-k + gates, K2 hist/scan/estimator
  csrc/kernels/expert_ffn.cu    K3 grouped SwiGLU expert FFN (TMA-staged), combine
  csrc/host/scheduler.*         HWB + AEE primitives (moesim operator API mirror)
  csrc/host/step_scheduler.*    two-phase verification-step scheduler
  csrc/host/engine.*            device engine (slot pools, copy streams, NCCL)
  csrc/abi.cpp                  extern "C" boundary = include/moespac/moespac.h

``abi`` is the ctypes binding of that boundary.
"""
from . import abi  # noqa: F401
from .configs import CONFIGS, WorkloadConfig  # noqa: F401

__all__ = ["abi", "CONFIGS", "WorkloadConfig"]
