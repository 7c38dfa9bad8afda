"""B200-native bulk ShaDow subgraph sampler (arXiv 2504.04670 hot path).

The product is native: lib/libhgs.so (CUDA kernels for sm_100a + the C ABI of
include/hgs.h) and lib/libhitgnn_gpu.so (the reference's C++ sampler API,
include/hitgnn/*.hpp, over that ABI). This package holds the in-tree build
(build.py), ctypes bindings (hgs.py), workload construction (workload.py) and
the multi-GPU shard rule (sharding.py).
"""
__all__ = ["hgs", "workload", "sharding", "build"]
