"""B200-native block-regression compressor hot path of SZ3 (arxiv 2111.02925).

The compute lives in ``libsz3g.so`` (csrc/, hand-written sm_100a CUDA behind the C ABI of
``include/sz3g.h``); ``sz3g`` is its ctypes binding and ``dist`` the slab sharding over ranks.
Importing this package does not load the library; the first call does, and fails loudly if the
library was not built.
"""
from .sz3g import (Compressed, CompressBuffers, SZ3GError, compress, decompress, histogram, load, num_blocks,
                   regression_compress, regression_decompress, value_range)

__all__ = ["Compressed", "CompressBuffers", "SZ3GError", "compress", "decompress", "histogram", "load", "num_blocks",
           "regression_compress", "regression_decompress", "value_range"]
