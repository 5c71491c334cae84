"""B200-native backend for the SpDISTAL hot path (arXiv 2207.13901).

The product is libspdistal_b200.so (C-ABI: include/spdistal_b200.h): device
storage, GPU dependent partitioning, sm_100a leaf kernels for SpMV, SpMM,
SDDMM, SpTTV, SpMTTKRP and SpAdd3, and the deterministic colour combine over
NCCL.  `host` mirrors the reference's interface over that ABI.
"""
__all__ = ["host"]
