"""Thin Python API over libspgemm.so — the same names as the C ABI (include/spgemm.h).

PyTorch provides device memory, streams and (for ``DistSpGEMM``) the process-group
bootstrap; every step of C = A·B runs in the library's CUDA kernels.  No computation
happens here: tensors are checked for dtype/device/contiguity and their pointers passed.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import (FLAG_INPUTS_REPLICATED, FLAG_PRECISE, FLAG_UPPER_BOUND, FLAG_VALIDATE,  # noqa: F401
                   SpgemmError, SpgemmStats, check, load)


@dataclass
class DeviceCsr:
    """CSR on a CUDA device: int64 row_ptr [rows+1], int32 col_idx [nnz], fp64 val [nnz]."""
    rows: int
    cols: int
    rp: torch.Tensor
    ci: torch.Tensor
    val: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.ci.numel())

    @staticmethod
    def from_host(M, device="cuda", pin: bool = False, dtype=torch.float64) -> "DeviceCsr":
        """Copy a host CSR (anything with .shape/.rp/.ci/.val numpy arrays) to the device;
        dtype=torch.float32 for SpSGEMM values."""
        def t(a, dt):
            x = torch.from_numpy(a).to(dt)
            if pin:
                x = x.pin_memory()
            return x.to(device, non_blocking=pin)
        return DeviceCsr(int(M.shape[0]), int(M.shape[1]), t(M.rp, torch.int64), t(M.ci, torch.int32),
                         t(M.val, dtype))

    def to_host(self):
        return (self.rp.cpu().numpy(), self.ci.cpu().numpy(), self.val.cpu().numpy())


def _ptr(t: torch.Tensor | None, dtype: torch.dtype, name: str) -> int | None:
    if t is None:
        return None
    if t.dtype != dtype:
        raise TypeError("%s must be %s, got %s" % (name, dtype, t.dtype))
    if not t.is_cuda:
        raise TypeError("%s must be a CUDA tensor" % name)
    if not t.is_contiguous():
        raise ValueError("%s must be contiguous" % name)
    return t.data_ptr() if t.numel() > 0 else None


def _csr_ptrs(M: DeviceCsr, name: str, vdtype=torch.float64):
    return (_ptr(M.rp, torch.int64, name + ".rp"), _ptr(M.ci, torch.int32, name + ".ci"),
            _ptr(M.val, vdtype, name + ".val"))


def _stream_handle(stream) -> int | None:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream or None


def set_debug(force_tier: int = -1, long_initial_capacity: int = 0, long_threshold: int = 0):
    """Testing knobs: force a stage-3 class, the initial long-row capacity, the long threshold."""
    lib = load()
    check(lib.spgemm_set_debug(force_tier, long_initial_capacity, long_threshold))


def set_debug_long_bucket(min_window: int = 0):
    """Test knob: long rows with column windows wider than `min_window` take the bucket path
    in precise numeric (0 = default 2^18, negative = never).  See spgemm_set_debug_long_bucket."""
    lib = load()
    check(lib.spgemm_set_debug_long_bucket(int(min_window)))


def set_debug_long_tile(tile_columns: int = 0):
    """Testing knob: long-row bitmap tiles of at most tile_columns columns (0 = default)."""
    lib = load()
    check(lib.spgemm_set_debug_long_tile(int(tile_columns)))


def trim_workspace_cache(keep_bytes: int = 0):
    """Return the library pool's cached device memory above keep_bytes."""
    lib = load()
    check(lib.spgemm_trim_workspace_cache(int(keep_bytes)))


def partition_rows(u_inclusive_scan, nranks: int):
    """Host partition rule of dist_symbolic (numpy int64 in, numpy int64 splits out)."""
    import numpy as np
    scan = np.ascontiguousarray(u_inclusive_scan, dtype=np.int64)
    out = np.zeros(nranks + 1, dtype=np.int64)
    lib = load()
    check(lib.spgemm_partition_rows(scan.ctypes.data if scan.size else None, scan.size, nranks,
                                    out.ctypes.data))
    return out


def _i64(a):
    import numpy as np
    return np.ascontiguousarray(a, dtype=np.int64)


def dist_block_entries(rp_at_splits):
    """Host protocol step: entry ranges [(begin, end)] of the row blocks from A.row_ptr at the splits."""
    import numpy as np
    x = _i64(rp_at_splits)
    out = np.zeros(2 * (x.size - 1), dtype=np.int64)
    check(load().spgemm_dist_block_entries(x.ctypes.data, x.size - 1, out.ctypes.data))
    return out.reshape(-1, 2)


def dist_slice_layout(row_begin, row_end, nnz, k: int):
    """Host protocol step: global entry offset of every B slice (+ nnz(B) last)."""
    import numpy as np
    rb, re_, nz = _i64(row_begin), _i64(row_end), _i64(nnz)
    out = np.zeros(rb.size + 1, dtype=np.int64)
    check(load().spgemm_dist_slice_layout(rb.ctypes.data, re_.ctypes.data, nz.ctypes.data, rb.size, k,
                                          out.ctypes.data))
    return out


def dist_offsets(local_nnz, rank: int):
    """Host protocol step: (global row-pointer offset of `rank`, nnz(C))."""
    x = _i64(local_nnz)
    off, tot = ctypes.c_int64(), ctypes.c_int64()
    check(load().spgemm_dist_offsets(x.ctypes.data, x.size, rank, ctypes.byref(off), ctypes.byref(tot)))
    return int(off.value), int(tot.value)


def debug_partition(u_scan_dev: torch.Tensor, nranks: int):
    """The device partition kernel of dist_symbolic on a device inclusive scan (test hook)."""
    import numpy as np
    out = np.zeros(nranks + 1, dtype=np.int64)
    check(load().spgemm_debug_partition(_ptr(u_scan_dev, torch.int64, "scan"), u_scan_dev.numel(), nranks,
                                        out.ctypes.data))
    return out


class SpGEMM:
    """One C = A·B multiplication: create → symbolic → numeric → destroy (C ABI names)."""

    def __init__(self, A: DeviceCsr, B: DeviceCsr, flags: int = 0, stream: torch.cuda.Stream | None = None):
        if A.cols != B.rows:
            raise ValueError("dimension mismatch: A is %dx%d, B is %dx%d" % (A.rows, A.cols, B.rows, B.cols))
        self.lib = load()
        self.A, self.B = A, B  # keep the inputs alive for the handle's lifetime
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.h = ctypes.c_void_p()
        self.f32 = A.val.dtype == torch.float32  # SpSGEMM (spgemm_create_f32)
        vdt = torch.float32 if self.f32 else torch.float64
        ap, bp = _csr_ptrs(A, "A", vdt), _csr_ptrs(B, "B", vdt)
        create = self.lib.spgemm_create_f32 if self.f32 else self.lib.spgemm_create
        check(create(ctypes.byref(self.h), A.rows, A.cols, B.cols, ap[0], ap[1], ap[2], A.nnz,
                     bp[0], bp[1], bp[2], B.nnz, _stream_handle(self.stream), flags))
        self.nnz_c = None

    def symbolic(self) -> int:
        n = ctypes.c_int64()
        check(self.lib.spgemm_symbolic(self.h, ctypes.byref(n)), self.h)
        self.nnz_c = int(n.value)
        return self.nnz_c

    def numeric(self, c_rp: torch.Tensor | None = None, c_ci: torch.Tensor | None = None,
                c_val: torch.Tensor | None = None):
        if self.nnz_c is None:
            raise SpgemmError(5, "numeric before symbolic")
        dev = self.A.rp.device
        vdt = torch.float32 if self.f32 else torch.float64
        if c_rp is None:
            c_rp = torch.empty(self.A.rows + 1, dtype=torch.int64, device=dev)
            c_ci = torch.empty(self.nnz_c, dtype=torch.int32, device=dev)
            c_val = torch.empty(self.nnz_c, dtype=vdt, device=dev)
        numeric = self.lib.spgemm_numeric_f32 if self.f32 else self.lib.spgemm_numeric
        check(numeric(self.h, _ptr(c_rp, torch.int64, "c_rp"), _ptr(c_ci, torch.int32, "c_ci"),
                      _ptr(c_val, vdt, "c_val")), self.h)
        return DeviceCsr(self.A.rows, self.B.cols, c_rp, c_ci, c_val)

    def stats(self) -> dict:
        s = SpgemmStats()
        check(self.lib.spgemm_get_stats(self.h, ctypes.byref(s)), self.h)
        return s.as_dict()

    def debug_u(self):
        dev = self.A.rp.device
        u = torch.empty(max(self.A.rows, 1), dtype=torch.int64, device=dev)
        t = torch.empty(max(self.A.rows, 1), dtype=torch.int32, device=dev)
        check(self.lib.spgemm_debug_get_u(self.h, u.data_ptr(), t.data_ptr()), self.h)
        return u[: self.A.rows], t[: self.A.rows]

    def destroy(self):
        if self.h:
            self.lib.spgemm_destroy(self.h)
            self.h = ctypes.c_void_p()

    close = destroy

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def spgemm(A: DeviceCsr, B: DeviceCsr, flags: int = 0, stream=None) -> DeviceCsr:
    """C = A·B through the four stages (convenience: allocates C with torch)."""
    op = SpGEMM(A, B, flags, stream)
    try:
        op.symbolic()
        return op.numeric()
    finally:
        op.destroy()


def nccl_unique_id() -> bytes:
    lib = load()
    buf = ctypes.create_string_buffer(128)
    check(lib.spgemm_nccl_get_unique_id(buf))
    return buf.raw


class DistSpGEMM:
    """Row-block multi-GPU C = A·B (one process per GPU).  The NCCL id is shipped with
    torch.distributed (any backend); all data movement is NCCL inside the library."""

    def __init__(self, rank: int, nranks: int, uid: bytes, m: int, k: int, n: int,
                 A: DeviceCsr | None, B: DeviceCsr | None, flags: int = 0, stream=None,
                 a_rows: tuple | None = None, b_rows: tuple | None = None):
        """a_rows / b_rows given: sharded inputs (spgemm_dist_create_sharded) — A holds this
        rank's rows a_rows = (begin, end) of the global A, B this rank's rows b_rows of B."""
        self.lib = load()
        self.A, self.B = A, B
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.h = ctypes.c_void_p()
        ap = _csr_ptrs(A, "A") if A is not None else (None, None, None)
        bp = _csr_ptrs(B, "B") if B is not None else (None, None, None)
        if a_rows is not None:
            check(self.lib.spgemm_dist_create_sharded(ctypes.byref(self.h), rank, nranks, uid, m, k, n, a_rows[0],
                                                      a_rows[1], ap[0], ap[1], ap[2], A.nnz, b_rows[0], b_rows[1],
                                                      bp[0], bp[1], bp[2], B.nnz, _stream_handle(self.stream),
                                                      flags))
        else:
            check(self.lib.spgemm_dist_create(ctypes.byref(self.h), rank, nranks, uid, m, k, n, ap[0], ap[1], ap[2],
                                              A.nnz if A is not None else 0, bp[0], bp[1], bp[2],
                                              B.nnz if B is not None else 0, _stream_handle(self.stream), flags))
        self.n = n
        self.block = None

    def symbolic(self):
        rb, re_, ln, gn = (ctypes.c_int64() for _ in range(4))
        check(self.lib.spgemm_dist_symbolic(self.h, ctypes.byref(rb), ctypes.byref(re_), ctypes.byref(ln),
                                            ctypes.byref(gn)), self.h)
        self.block = (int(rb.value), int(re_.value), int(ln.value), int(gn.value))
        return self.block

    def numeric(self, device="cuda"):
        rb, re_, ln, _ = self.block
        c_rp = torch.empty(re_ - rb + 1, dtype=torch.int64, device=device)
        c_ci = torch.empty(ln, dtype=torch.int32, device=device)
        c_val = torch.empty(ln, dtype=torch.float64, device=device)
        check(self.lib.spgemm_dist_numeric(self.h, c_rp.data_ptr(), _ptr(c_ci, torch.int32, "c_ci"),
                                           _ptr(c_val, torch.float64, "c_val")), self.h)
        return DeviceCsr(re_ - rb, self.n, c_rp, c_ci, c_val)

    def stats(self) -> dict:
        s = SpgemmStats()
        check(self.lib.spgemm_get_stats(self.h, ctypes.byref(s)), self.h)
        return s.as_dict()

    def destroy(self):
        if self.h:
            self.lib.spgemm_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass
