"""abin -- B200-native local adaptive binarization (arXiv 1905.13038 hot path).

The product is libabin.so (CUDA kernels for sm_100a behind a C ABI, see
include/abin.h); this package is its thin Python binding plus the multi-GPU
driver.  Import fails loudly when the CUDA library has not been built.
"""
from . import abin  # noqa: F401  (raises ImportError if libabin.so is missing)
from .abin import (bernsen, binarize_band, binarize_batched, binarize_rule, global_min, max_s, niblack, otsu,  # noqa: F401
                   probe_filter, quantile, sauvola, stats, version, wolf, wolf_adaptive)
