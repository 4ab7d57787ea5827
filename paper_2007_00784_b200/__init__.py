"""B200-native K-FAC preconditioner hot path (arXiv 2007.00784).

libkfac.so (csrc/, C-ABI in include/kfac.h) holds every kernel; `_lib` is the
ctypes binding and `preconditioner.KFACPreconditioner` the multi-GPU
orchestration.  Importing the package does not load CUDA; `import
paper_2007_00784_b200._lib` loads the library and fails loudly if it is missing.
"""
__all__ = ["lib"]


def lib():
    from . import _lib
    return _lib
