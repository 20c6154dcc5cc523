"""CPU oracle for C = A·B (CSR, fp64) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  The product package
``paper_1504_05022_b200`` never imports it and shares no code with it.

The arithmetic lives in ``oracle/oracle.cpp`` (plain C++/OpenMP, no FMA); this module
only builds it with g++ and marshals numpy arrays.  See the header of oracle.cpp for
which passage of PAPER.md each function follows:

* ``upper_bound``  — Algorithm "first stage" [P:198-212]
* ``bins``         — Algorithm "second stage" [P:226-260] (38 bins, hybrid C~ sizes [P:224])
* ``spgemm``       — Algorithm "Pseudocode for the SpGEMM" [P:115-138] with the dense SPA [P:142]

Parity pins: every function here is pinned by tests/test_oracle.py against values
that do not come from this code (dense brute force, closed forms, paper/SPEC worked
examples); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

I64P = ctypes.POINTER(ctypes.c_int64)
I32P = ctypes.POINTER(ctypes.c_int32)
F64P = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile oracle.cpp → liboracle.so (g++ -O3 -fopenmp -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O3", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_validate_csr.restype = ctypes.c_int
        lib.oracle_validate_csr.argtypes = [ctypes.c_int64, ctypes.c_int64, I64P, I32P, ctypes.c_int64]
        lib.oracle_upper_bound.restype = ctypes.c_int64
        lib.oracle_upper_bound.argtypes = [ctypes.c_int64, ctypes.c_int64, I64P, I32P, I64P, I64P]
        lib.oracle_bins.restype = ctypes.c_int64
        lib.oracle_bins.argtypes = [ctypes.c_int64, I64P, I32P, I64P]
        lib.oracle_spgemm_count.restype = ctypes.c_int64
        lib.oracle_spgemm_count.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, I64P, I32P,
                                            I64P, I32P, I64P, ctypes.c_int]
        lib.oracle_spgemm_fill.restype = None
        lib.oracle_spgemm_fill.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, I64P, I32P, F64P,
                                           I64P, I32P, F64P, I64P, I32P, F64P, F64P, ctypes.c_int]
        F32P = ctypes.POINTER(ctypes.c_float)
        lib.oracle_spgemm_fill_f32.restype = None
        lib.oracle_spgemm_fill_f32.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, I64P, I32P, F32P,
                                               I64P, I32P, F32P, I64P, I32P, F32P, F64P, ctypes.c_int]
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ct)


def _csr(rp, ci, val=None):
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    if val is None:
        return rp, ci
    return rp, ci, np.ascontiguousarray(val, dtype=np.float64)


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def validate_csr(rows: int, cols: int, rp, ci) -> int:
    """0 if the CSR invariants hold, else an error code (see oracle.cpp)."""
    rp, ci = _csr(rp, ci)
    if rp.shape[0] != rows + 1:
        return 3
    return int(_load().oracle_validate_csr(rows, cols, _p(rp, I64P), _p(ci, I32P), ci.shape[0]))


def upper_bound(A, B, r0: int = 0, r1: int | None = None):
    """Stage 1 [P:198-212]: (u[r0:r1], sum u)."""
    m = A.shape[0]
    r1 = m if r1 is None else r1
    arp, aci = _csr(A.rp, A.ci)
    brp, _ = _csr(B.rp, B.ci)
    u = np.empty(max(r1 - r0, 0), dtype=np.int64)
    tot = _load().oracle_upper_bound(r0, r1, _p(arp, I64P), _p(aci, I32P), _p(brp, I64P), _p(u, I64P))
    return u, int(tot)


def bins(u):
    """Stage 2 [P:226-260]: (bin[m] in 0..37, ctil_nnz[m], nnz(C~))."""
    u = np.ascontiguousarray(u, dtype=np.int64)
    b = np.empty(u.shape[0], dtype=np.int32)
    c = np.empty(u.shape[0], dtype=np.int64)
    tot = _load().oracle_bins(u.shape[0], _p(u, I64P), _p(b, I32P), _p(c, I64P))
    return b, c, int(tot)


@dataclass
class OracleResult:
    rp: np.ndarray      # int64 [rows+1], relative to row r0 (rp[0] == 0)
    ci: np.ndarray      # int32 [nnz]
    val: np.ndarray     # float64 [nnz]
    bound: np.ndarray | None  # float64 [nnz]: sum_j |a_ij||b_jk| (tolerance scale)
    r0: int = 0


def spgemm(A, B, r0: int = 0, r1: int | None = None, with_bound: bool = True,
           threads: int = 0, fp32: bool = False) -> OracleResult:
    """C[r0:r1] = A[r0:r1]·B by row-wise Gustavson + dense SPA [P:115-138], [P:142].
    fp32: SpSGEMM — A's and B's values taken as float32, products and sums in float32
    (the result's val is float32)."""
    if A.shape[1] != B.shape[0]:
        raise ValueError("dimension mismatch: A is %dx%d, B is %dx%d" % (A.shape + B.shape))
    m, n = A.shape[0], B.shape[1]
    r1 = m if r1 is None else r1
    lib = _load()
    arp, aci, aval = _csr(A.rp, A.ci, A.val)
    brp, bci, bval = _csr(B.rp, B.ci, B.val)
    rows = max(r1 - r0, 0)
    nnz_row = np.empty(rows, dtype=np.int64)
    lib.oracle_spgemm_count(r0, r1, n, _p(arp, I64P), _p(aci, I32P), _p(brp, I64P), _p(bci, I32P),
                            _p(nnz_row, I64P), threads)
    crp = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(nnz_row, out=crp[1:])
    nnz = int(crp[-1])
    cci = np.empty(nnz, dtype=np.int32)
    bound = np.empty(nnz, dtype=np.float64) if with_bound else None
    if fp32:
        F32P = ctypes.POINTER(ctypes.c_float)
        a32 = np.ascontiguousarray(A.val, dtype=np.float32)
        b32 = np.ascontiguousarray(B.val, dtype=np.float32)
        cval = np.empty(nnz, dtype=np.float32)
        lib.oracle_spgemm_fill_f32(r0, r1, n, _p(arp, I64P), _p(aci, I32P), _p(a32, F32P), _p(brp, I64P),
                                   _p(bci, I32P), _p(b32, F32P), _p(crp, I64P), _p(cci, I32P), _p(cval, F32P),
                                   _p(bound, F64P) if bound is not None else None, threads)
        return OracleResult(crp, cci, cval, bound, r0)
    cval = np.empty(nnz, dtype=np.float64)
    lib.oracle_spgemm_fill(r0, r1, n, _p(arp, I64P), _p(aci, I32P), _p(aval, F64P), _p(brp, I64P),
                           _p(bci, I32P), _p(bval, F64P), _p(crp, I64P), _p(cci, I32P), _p(cval, F64P),
                           _p(bound, F64P) if bound is not None else None, threads)
    return OracleResult(crp, cci, cval, bound, r0)
