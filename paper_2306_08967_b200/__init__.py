"""B200-native (sm_100a) DAMF dynamic-embedding hot path.

The product is libdamf_gpu.so (C ABI: include/damf_gpu.h); `engine` is its
Python binding and `workloads` builds the seeded synthetic inputs of the five
BASELINE configurations.
"""
from . import workloads  # noqa: F401  (pure numpy input generation)

__all__ = ["engine", "workloads"]
