"""B200-native (sm_100a) implicit-integration hot path of P-Cloth
(arXiv 2008.00409): dynamic 3x3-block assembly, partitioned block-Jacobi
PCG, spatial-hash broad phase. The compute lives in libweft_gpu.so (C-ABI:
include/weft_gpu.h); `weft` is the Python mirror of the reference interface."""

__all__ = ["weft", "build"]
