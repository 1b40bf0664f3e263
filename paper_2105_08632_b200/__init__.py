"""B200-native SDRT residual / RK4 hot path (arXiv 2105.08632).

The product is libsdrt.so (C ABI, include/sdrt.h): host setup in C++ (__float128
operators, pattern-mesh tables) and sm_100a CUDA kernels.  ``sdrt`` is a thin
ctypes binding; ``solver`` wraps it with torch-owned device memory.
"""
