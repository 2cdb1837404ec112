"""spmvcomp-b200: B200-native SpMV path of arxiv 1612.00530 (`spmvcomp`).

Importing this package loads the CUDA library (libspmvcomp_b200.so); there is no
CPU fallback and the import fails loudly when the library has not been built.
"""
from . import _cabi  # noqa: F401  (raises ImportError when the .so is missing)
from .api import *  # noqa: F401,F403
from .api import DeviceMatrix, DeviceVector, GridSpec  # noqa: F401
from .slab import DeviceSlabSpmv, SlabCg, SlabLayout, SlabSpmv, build_slab_pattern, merge_dictionaries  # noqa: F401,E402
