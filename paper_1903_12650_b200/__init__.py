"""B200-native LARS gradient-combine-and-update library (arxiv 1903.12650 hot path).

The product is the C-ABI shared library ``liblars_b200.so`` (include/lars.h); this package holds its
CUDA/C++ sources (``csrc/``), the build script and a thin ctypes binding (``lars``).
"""
from .lars import (DTYPE, KIND, Lars, LarsError, LarsLibraryMissing, declared_functions, default_hparams,
                   get_unique_id, lars_init, load_library)

__all__ = ["DTYPE", "KIND", "Lars", "LarsError", "LarsLibraryMissing", "declared_functions", "default_hparams",
           "get_unique_id", "lars_init", "load_library"]
