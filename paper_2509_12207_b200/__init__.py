"""B200-native batched simulation of UrgenGo's urgency-aware kernel-launch policy.

The product path is liburg.so (CUDA for sm_100a, C ABI in include/urg.h) and the
thin ctypes binding in ``urg``; ``dist`` shards scenarios over GPUs.
"""
from .urg import DeviceWorkload, UrgError, lib  # noqa: F401
