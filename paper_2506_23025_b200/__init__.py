"""paper_2506_23025_b200 -- the TriRun ternary-linear hot path, B200-native.

Keeps the reference package's (`tritpack`) pack/unpack and ternary-linear API
(DType, BLOCK_ELEMENTS, pack_matrix, PackedMatrix, gemm, gemv,
dequantize_matrix, gemv_reference, quantize_rows, dequantize_rows, backend
selection) and adds the GPU fast path (TernaryWeight, linear, TernaryLinear).
All compute runs in libtritrun.so (hand-written sm_100a CUDA behind a C-ABI).
"""

from .backend import available as available_backends
from .backend import default_name as default_backend
from .blocks import (
    BLOCK_ELEMENTS,
    DType,
    QuantizationError,
    TernarizeResult,
    TQ1Block,
    TQ2Block,
    dequantize_block_tq1,
    dequantize_block_tq2,
    dequantize_rows,
    quantize_block_tq1,
    quantize_block_tq2,
    quantize_rows,
    ternarize,
)
from .device import TernaryLinear, TernaryWeight, linear
from .packed_linear import PackedMatrix, dequantize_matrix, gemm, gemv, gemv_reference, pack_matrix
from .perf import BenchRow, bench, critical_batch

__version__ = "0.1.0"

__all__ = [
    "available_backends", "default_backend", "BLOCK_ELEMENTS", "DType", "QuantizationError", "TernarizeResult",
    "TQ1Block", "TQ2Block", "dequantize_block_tq1", "dequantize_block_tq2", "dequantize_rows",
    "quantize_block_tq1", "quantize_block_tq2", "quantize_rows", "ternarize", "TernaryLinear", "TernaryWeight",
    "linear", "PackedMatrix", "dequantize_matrix", "gemm", "gemv", "gemv_reference", "pack_matrix", "BenchRow",
    "bench", "critical_batch", "__version__",
]
