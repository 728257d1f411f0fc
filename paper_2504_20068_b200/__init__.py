"""B200-native JITServe GMAX scheduling step (arXiv 2504.20068).

The hot path is libjitsched.so (hand-written CUDA for sm_100a behind the C ABI in
include/jit_sched.h); ``jitsched`` is its ctypes binding.  There is no CPU fallback.
"""
from .jitsched import Scheduler, JitSchedError, load_library, LIB_PATH  # noqa: F401

__all__ = ["Scheduler", "JitSchedError", "load_library", "LIB_PATH"]
