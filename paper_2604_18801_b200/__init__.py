"""B200-native FoF-connectivity correction for error-bounded lossy particle compression
(arXiv 2604.18801).  Thin Python binding over ``libcc.so`` (include/cc.h): argument
marshalling only -- every step of the path runs in the CUDA kernels of ``csrc/``.  PyTorch
provides device memory, streams and process groups.  There is no CPU fallback: importing
works without a GPU (for building and ABI checks) but every compute call needs the CUDA
extension and a device, and raises otherwise.
"""
from .binding import (CC_CORR, CC_DECOMP, CC_ORIG, CCError, Corrector, Params, STOP_ACTIVE, STOP_EPS, VGroup,
                      STOP_NONE, STOP_RESTORED, hmf, lib, lib_path, nccl_unique_id, shell_masks, slab_of)

__all__ = ["Corrector", "Params", "VGroup", "CCError", "hmf", "lib", "lib_path", "nccl_unique_id", "slab_of", "CC_ORIG",
           "CC_DECOMP", "CC_CORR", "STOP_ACTIVE", "STOP_EPS", "STOP_NONE", "STOP_RESTORED"]
