"""roundpipe-b200: a B200-native RoundPipe training step (arXiv 2604.27085).

Layers:
  planner  — the reference planner API (partition / dispatch / timeline /
             LPT windows / consistency protocol) over the C-ABI;
  kernels  — sm_100a kernels of one stage (ctypes over include/rp/kernels.h);
  runtime  — the C++ executor walking the dispatch list on B200s.
All compute goes through libroundpipe_b200.so; nothing here falls back to
PyTorch or the CPU.
"""
from ._native import (NativeError, InputError, InfeasibleError,  # noqa: F401
                      ProtocolViolation, CapExceededError, CudaError)

__all__ = ["planner", "kernels", "runtime"]
