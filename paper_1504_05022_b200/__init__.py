"""B200-native four-stage CSR SpGEMM (Liu & Vinter, arXiv 1504.05022).

The computation lives in libspgemm.so (csrc/, CUDA for sm_100a, C ABI in
include/spgemm.h).  This package only builds and binds it; importing the API raises if
the library is missing — there is no Python or CPU fallback.
"""
from .spgemm import (FLAG_INPUTS_REPLICATED, FLAG_PRECISE, FLAG_UPPER_BOUND, FLAG_VALIDATE,  # noqa: F401
                     DeviceCsr, DistSpGEMM, SpGEMM, SpgemmError, nccl_unique_id, partition_rows,
                     set_debug, set_debug_long_bucket, set_debug_long_tile, spgemm, trim_workspace_cache, dist_block_entries,
                     dist_slice_layout, dist_offsets, debug_partition)
from ._lib import LIB_PATH, TIER_NAMES, load  # noqa: F401
