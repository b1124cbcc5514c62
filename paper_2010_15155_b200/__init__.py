"""B200-native Kernel Aggregated FMM (arXiv 2010.15155), evaluation pass.

The compute path is libkafmm.so (hand-written CUDA for sm_100a behind the C
ABI in include/kafmm.h); this package is a thin ctypes binding with the same
names.  There is no CPU fallback: if the library or a CUDA device is missing,
every call raises.
"""
from .kafmm import (KERNELS, KAFMM, KAFMM2, KAFMMWall, DistKAFMM, KafmmError, Info, kernel_dims, lib_path,
                    load_library)

__all__ = ["KERNELS", "KAFMM", "KAFMM2", "KAFMMWall", "DistKAFMM", "KafmmError", "Info", "kernel_dims", "lib_path", "load_library"]
