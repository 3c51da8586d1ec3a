"""B200-native reuse-prefill hot path of PCR (arXiv 2603.23049).

The product is libpcr.so (include/pcr.h): C++ host control (prefix tree + look-ahead LRU)
and hand-written sm_100a kernels (16-byte host->HBM gather, suffix append, tcgen05/TMEM/TMA
suffix attention), driven per layer on two CUDA streams.  `pcr` is the ctypes binding.
"""
from .pcr import (MODE_ONLY_DOWN, MODE_ONLY_UP, MODE_OVERLAP, MODE_SYNC, SHARD_CONTEXT, SHARD_HEADS, Context,  # noqa: F401
                  PcrError, blake2b, comm_unique_id,
                  load_library)
