"""B200-native hot path of the neural path tracer of arXiv 2305.20061.

Layout: csrc/ (CUDA sm_100a kernels + C++ host runtime behind include/pt.h), pt.py (ctypes binding),
scenes.py (seeded synthetic inputs), dist.py (sample-partitioned multi-GPU rendering)."""
__all__ = ["pt", "scenes"]
