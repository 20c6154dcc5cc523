"""ctypes declarations for libspgemm.so (include/spgemm.h).  Argument marshalling only.

There is no fallback: if the shared library is missing this raises, it never computes
anything in Python.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# SPGEMM_LIB: an alternative in-tree build (A/B timing during development); default libspgemm.so
LIB_PATH = os.path.join(PKG, os.environ.get("SPGEMM_LIB", "libspgemm.so"))
NUM_TIERS = 21

TIER_NAMES = ["empty", "g1", "g2", "g4", "g8", "g16", "g32", "w64", "w128", "w256", "w512", "w1024",
              "w2048", "c2048", "c4096", "c8192", "e2048", "e4096", "e8192", "bw", "long"]

STATUS = {
    0: "SPGEMM_SUCCESS", 1: "SPGEMM_ERROR_INVALID_VALUE", 2: "SPGEMM_ERROR_INVALID_CSR",
    3: "SPGEMM_ERROR_INDEX_OVERFLOW", 4: "SPGEMM_ERROR_OUT_OF_MEMORY", 5: "SPGEMM_ERROR_INVALID_STATE",
    6: "SPGEMM_ERROR_CUDA", 7: "SPGEMM_ERROR_NCCL", 8: "SPGEMM_ERROR_INTERNAL",
}

FLAG_VALIDATE = 1 << 0
FLAG_INPUTS_REPLICATED = 1 << 1
FLAG_PRECISE = 1 << 2
FLAG_UPPER_BOUND = 1 << 3
FLAG_FP32 = 1 << 4


class SpgemmStats(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64), ("k", ctypes.c_int64), ("n", ctypes.c_int64),
        ("nnz_a", ctypes.c_int64), ("nnz_b", ctypes.c_int64),
        ("sum_u", ctypes.c_int64), ("nnz_c", ctypes.c_int64), ("max_u", ctypes.c_int64),
        ("tier_rows", ctypes.c_int64 * NUM_TIERS),
        ("ctil_entries", ctypes.c_int64), ("long_rows", ctypes.c_int64),
        ("long_entries", ctypes.c_int64), ("growth_rounds", ctypes.c_int32),
        ("flags", ctypes.c_int32), ("workspace_bytes", ctypes.c_int64),
        ("stage_ms", ctypes.c_float * 4),
        ("tier_ms", ctypes.c_float * NUM_TIERS),
        ("tier_a_entries", ctypes.c_int64 * NUM_TIERS),
        ("tier_products", ctypes.c_int64 * NUM_TIERS),
        ("tier_c_entries", ctypes.c_int64 * NUM_TIERS),
        ("launches_symbolic", ctypes.c_int32),
        ("launches_numeric", ctypes.c_int32),
        ("tier_ms_symbolic", ctypes.c_float * NUM_TIERS),
    ]

    def as_dict(self) -> dict:
        arrays = ("tier_rows", "stage_ms", "tier_ms", "tier_ms_symbolic", "tier_a_entries", "tier_products", "tier_c_entries")
        d = {f: getattr(self, f) for f, _ in self._fields_ if f not in arrays}
        d["tier_rows"] = {TIER_NAMES[t]: int(self.tier_rows[t]) for t in range(NUM_TIERS) if self.tier_rows[t]}
        d["stage_ms"] = [float(x) for x in self.stage_ms]
        d["classes"] = {TIER_NAMES[t]: dict(rows=int(self.tier_rows[t]), ms=float(self.tier_ms[t]),
                                            ms_symbolic=float(self.tier_ms_symbolic[t]),
                                            a_entries=int(self.tier_a_entries[t]),
                                            products=int(self.tier_products[t]),
                                            c_entries=int(self.tier_c_entries[t]))
                        for t in range(NUM_TIERS) if self.tier_rows[t]}
        return d


class SpgemmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


_lib = None
H = ctypes.c_void_p
P = ctypes.c_void_p
I64 = ctypes.c_int64


class _Tolerant:
    """Attribute access on an older in-tree build: missing entry points become no-op holders."""

    def __init__(self, lib):
        object.__setattr__(self, "_lib", lib)

    def __getattr__(self, name):
        try:
            return getattr(self._lib, name)
        except AttributeError:
            class _Missing:
                pass
            m = _Missing()
            object.__setattr__(self, name, m)
            return m

    def __setattr__(self, name, value):
        setattr(self._lib, name, value)


def load():
    """Load libspgemm.so (build it with `python -m paper_1504_05022_b200.build`)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("libspgemm.so is not built (%s); run `python -m paper_1504_05022_b200.build`"
                          % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    if os.environ.get("SPGEMM_LIB"):
        lib = _Tolerant(lib)  # development A/B builds may predate some entry points
    st = ctypes.c_int
    lib.spgemm_create.restype = st
    lib.spgemm_create.argtypes = [ctypes.POINTER(H), I64, I64, I64, P, P, P, I64, P, P, P, I64, P, ctypes.c_uint32]
    lib.spgemm_create_f32.restype = st
    lib.spgemm_create_f32.argtypes = [ctypes.POINTER(H), I64, I64, I64, P, P, P, I64, P, P, P, I64, P, ctypes.c_uint32]
    lib.spgemm_numeric_f32.restype = st
    lib.spgemm_numeric_f32.argtypes = [H, P, P, P]
    lib.spgemm_symbolic.restype = st
    lib.spgemm_symbolic.argtypes = [H, ctypes.POINTER(I64)]
    lib.spgemm_numeric.restype = st
    lib.spgemm_numeric.argtypes = [H, P, P, P]
    lib.spgemm_destroy.restype = st
    lib.spgemm_destroy.argtypes = [H]
    lib.spgemm_get_stats.restype = st
    lib.spgemm_get_stats.argtypes = [H, ctypes.POINTER(SpgemmStats)]
    lib.spgemm_debug_get_u.restype = st
    lib.spgemm_debug_get_u.argtypes = [H, P, P]
    lib.spgemm_set_debug.restype = st
    lib.spgemm_set_debug.argtypes = [ctypes.c_int32, I64, I64]
    lib.spgemm_set_debug_long_tile.restype = st
    lib.spgemm_set_debug_long_tile.argtypes = [I64]
    lib.spgemm_set_debug_long_bucket.restype = st
    lib.spgemm_set_debug_long_bucket.argtypes = [I64]
    lib.spgemm_trim_workspace_cache.restype = st
    lib.spgemm_trim_workspace_cache.argtypes = [I64]
    lib.spgemm_status_string.restype = ctypes.c_char_p
    lib.spgemm_status_string.argtypes = [st]
    lib.spgemm_last_error.restype = ctypes.c_char_p
    lib.spgemm_last_error.argtypes = [H]
    lib.spgemm_version.restype = ctypes.c_char_p
    lib.spgemm_version.argtypes = []
    lib.spgemm_nccl_get_unique_id.restype = st
    lib.spgemm_nccl_get_unique_id.argtypes = [ctypes.c_char_p]
    lib.spgemm_dist_create.restype = st
    lib.spgemm_dist_create.argtypes = [ctypes.POINTER(H), ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                       I64, I64, I64, P, P, P, I64, P, P, P, I64, P, ctypes.c_uint32]
    lib.spgemm_dist_symbolic.restype = st
    lib.spgemm_dist_symbolic.argtypes = [H, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64),
                                         ctypes.POINTER(I64)]
    lib.spgemm_dist_numeric.restype = st
    lib.spgemm_dist_numeric.argtypes = [H, P, P, P]
    lib.spgemm_dist_create_sharded.restype = st
    lib.spgemm_dist_create_sharded.argtypes = [ctypes.POINTER(H), ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                               I64, I64, I64, I64, I64, P, P, P, I64, I64, I64, P, P, P, I64, P,
                                               ctypes.c_uint32]
    lib.spgemm_partition_rows.restype = st
    lib.spgemm_partition_rows.argtypes = [P, I64, ctypes.c_int, P]
    lib.spgemm_dist_block_entries.restype = st
    lib.spgemm_dist_block_entries.argtypes = [P, ctypes.c_int, P]
    lib.spgemm_dist_slice_layout.restype = st
    lib.spgemm_dist_slice_layout.argtypes = [P, P, P, ctypes.c_int, I64, P]
    lib.spgemm_dist_offsets.restype = st
    lib.spgemm_dist_offsets.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(I64), ctypes.POINTER(I64)]
    lib.spgemm_debug_partition.restype = st
    lib.spgemm_debug_partition.argtypes = [P, I64, ctypes.c_int, P]
    _lib = lib
    return lib


def check(status: int, handle=None):
    if status != 0:
        lib = load()
        msg = lib.spgemm_last_error(handle).decode(errors="replace")
        raise SpgemmError(status, msg)
