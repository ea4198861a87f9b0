"""B200-native batched TFHE gate bootstrapping behind CryptoEmu's Backend seam.

The product is ``_lib/libcvm_b200.so`` (CUDA sm_100a kernels + C++ host side,
C ABI in ``include/cvm_gpu.h``); this package is a thin ctypes front end.
"""
from ._native import (CvmDeviceError, CvmError, CvmInputError, CvmStateError,  # noqa: F401
                      LWE_WORDS, LIB_PATH)
from .api import (FU, FU_OPS, KIND, OPCODE, Backend, Context, KeySet,  # noqa: F401
                  fu_batch)
