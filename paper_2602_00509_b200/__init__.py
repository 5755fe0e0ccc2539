"""B200-native PROBE expert-parallel MoE hot path (arXiv 2602.00509).

The product is libprobe.so (C-ABI in include/probe.h, sm_100a CUDA kernels);
this package only builds it and marshals arguments.
"""
from ._lib import LIB_PATH, ProbeError, load  # noqa: F401
from .runtime import ProbeConfig, ProbeRuntime, bench_gemm, test_gemm, workspace_sizes  # noqa: F401
