"""B200-native Tofu hot path (arXiv 1807.08887): libtofu.so (C ABI, sm_100a
kernels + C++ planner/executor) and its ctypes binding ``tofu``."""
from . import tofu  # noqa: F401
