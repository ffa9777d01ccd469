"""B200-native dynamic volume lines (arXiv 2306.11612): the data-parallel hot path.

The compute lives in the sm_100a CUDA library ``libdvl.so`` (csrc/, C ABI in
include/dvl.h); this package is its thin Python binding.
"""
from .dvl import (Context, DvlError, LocalGroup, VERTEX_DTYPE, hilbert_encode_host,  # noqa: F401
                  hilbert_states, load, LIB_PATH, SYMBOLS, select_splitters)
