"""B200-native batched TFHE gate bootstrapping behind CryptoEmu's Backend seam.

The product is ``_lib/libcvm_b200.so`` (CUDA sm_100a kernels + C++ host side,
C ABI in ``include/cvm_gpu.h``); this package is a thin ctypes front end.
"""
from ._native import (CvmDeviceError, CvmError, CvmInputError, CvmStateError,  # noqa: F401
                      LWE_WORDS, LIB_PATH)
from .api import (DAG_DTYPE, KIND, Backend, Context, Dag, KeySet,  # noqa: F401
                  dag_batch)
