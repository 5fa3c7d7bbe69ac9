"""B200-native gradient-compression engine (drop-in for the `gradcomp` reference path).

compress -> aggregate -> decompress with error feedback for THC (rotated stochastic
quantization with partial rotation and saturation), TopK / TopK-Chunked and PowerSGD,
plus the dense FP16 / FP32 baselines, as sm_100a CUDA kernels behind the C ABI in
include/gradcomp_b200.h (libgradcomp_b200.so).  Public names mirror gradcomp's
(pkg/src/gradcomp/__init__.py:15-51).
"""

__version__ = "0.1.0"

from . import _native
from .configs import (
    ChunkedTopKConfig, CompressorConfig, DegenerateMatrixError, DenseConfig, PowerSgdConfig, RotatedQuantConfig,
    TopKConfig, chunks_for_budget, matrix_shape_for, scheme_label, topk_for_budget,
)
from .ledger import OverflowStats, TrafficLedger, WorkerGroup, overflow_rate
from .vectors import ChunkGeometry, GradientVector, SeedSpec, fnv1a64, next_pow2, pad_to_pow2, splitmix64

_native.lib()  # fail loudly at import if the native library is missing

from .pipeline import (  # noqa: E402
    GradientPipeline, RoundResult, make_pipeline, run_chunked_topk_round, run_dense_round, run_powersgd_round,
    run_rotated_quant_round, run_topk_round,
)

__all__ = [
    "ChunkGeometry", "ChunkedTopKConfig", "CompressorConfig", "DegenerateMatrixError", "DenseConfig",
    "GradientPipeline", "GradientVector", "OverflowStats", "PowerSgdConfig", "RotatedQuantConfig", "RoundResult",
    "SeedSpec", "TopKConfig", "TrafficLedger", "WorkerGroup", "chunks_for_budget", "fnv1a64", "make_pipeline",
    "matrix_shape_for", "next_pow2", "overflow_rate", "pad_to_pow2", "run_chunked_topk_round", "run_dense_round",
    "run_powersgd_round", "run_rotated_quant_round", "run_topk_round", "scheme_label", "splitmix64",
    "topk_for_budget",
]
