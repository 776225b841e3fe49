"""B200-native weak-admissibility H-matrix-vector product (arXiv 2008.12441).

The product is libhmat.so (C ABI in include/hmat.h, sm_100a kernels in csrc/);
`hmat` is its thin ctypes binding.
"""
from . import hmat  # noqa: F401
from .hmat import HMatrix, HMatError  # noqa: F401
