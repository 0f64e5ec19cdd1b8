"""paper_2104_14129_b200 -- B200-native ActNN activation compressor (arXiv 2104.14129).

The hot path (per-group stochastic-rounding quantiser + bit packer, its
unpacker/dequantiser and the greedy per-sample bit allocator) runs in
hand-written sm_100a CUDA kernels behind the C-ABI in ``include/actnn.h``
(``libactnn.so``).  This package is the thin Python binding over that ABI:
argument marshalling only.  There is no CPU fallback: every entry point raises
if the CUDA library or a GPU is missing.
"""
from .api import (  # noqa: F401
    ActnnError, LayerAllocator, Packed, abi_version, allocate_bits, allocate_layers, compress,
    decompress, dequantize, grad_sqnorm, gradmag_ema, gradmag_gather, gradmag_scatter,
    group_stats, library_path, maxpool2d, maxpool2d_backward, packed_bytes, quantize,
    relu_backward, relu_pack, uniform_bits,
)
