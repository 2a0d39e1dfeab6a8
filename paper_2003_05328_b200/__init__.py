"""B200-native (sm_100a) ENSEI oblivious frequency-domain convolution hot path.

The product is libensei_gpu.so (CUDA kernels + the C ABI of include/ensei_gpu.h);
this package holds its sources (csrc/), the in-tree build recipe (build.py) and
the Python mirror of the reference operator API (ops.py, protocol.py).
"""
from ._lib import EnseiError, lib  # noqa: F401
