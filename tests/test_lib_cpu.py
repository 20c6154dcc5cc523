"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/spgemm.h
declares, and its host-only logic (status strings, argument errors, partition rule)
behaves — no kernel is launched here."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1504_05022_b200 as sg
from paper_1504_05022_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "spgemm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spgemm_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), "libspgemm.so does not export %s" % s


def test_version_and_status_strings():
    lib = _lib.load()
    assert b"sm_100a" in lib.spgemm_version()
    for code, name in _lib.STATUS.items():
        assert lib.spgemm_status_string(code).decode() == name


def test_create_argument_errors_without_gpu():
    lib = _lib.load()
    h = ctypes.c_void_p()
    # negative size → INVALID_VALUE before any device call
    assert lib.spgemm_create(ctypes.byref(h), -1, 1, 1, 1, None, None, 0, 1, None, None, 0, None, 0) == 1
    # m > INT32_MAX → INDEX_OVERFLOW
    assert lib.spgemm_create(ctypes.byref(h), 1 << 31, 1, 1, 1, None, None, 0, 1, None, None, 0, None, 0) == 3
    # unknown flag bits
    assert lib.spgemm_create(ctypes.byref(h), 1, 1, 1, 1, None, None, 0, 1, None, None, 0, None, 1 << 9) == 1
    assert b"unknown flag" in lib.spgemm_last_error(None)
    # NULL handle out-pointer
    assert lib.spgemm_create(None, 1, 1, 1, 1, None, None, 0, 1, None, None, 0, None, 0) == 1
    assert lib.spgemm_destroy(None) == 0
    n = ctypes.c_int64()
    assert lib.spgemm_symbolic(None, ctypes.byref(n)) == 1
    assert lib.spgemm_numeric(None, None, None, None) == 1


def _split_ref(scan, P):
    """Plain restatement of the rule s_r = min{i : scan[i] >= ceil(r·total/P)} + 1."""
    m = len(scan)
    total = int(scan[-1]) if m else 0
    out = [0]
    for r in range(1, P):
        t = -(-r * total // P)
        if t == 0:
            s = 0
        else:
            idx = next((i for i in range(m) if scan[i] >= t), m)
            s = min(idx + 1, m)
        out.append(max(s, out[-1]))
    out.append(m)
    return out


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_partition_rule(P, seed):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, 50, size=200)
    u[rng.integers(0, 200, size=5)] = rng.integers(500, 5000, size=5)  # a few heavy rows
    scan = np.cumsum(u)
    s = sg.partition_rows(scan, P)
    assert s.tolist() == _split_ref(scan.tolist(), P)
    assert s[0] == 0 and s[-1] == 200 and np.all(np.diff(s) >= 0)
    # balance: each block's products within max(u) of Σu/P (the stated ±max u_i bound)
    tot = scan[-1]
    for r in range(P):
        a = scan[s[r] - 1] if s[r] > 0 else 0
        b = scan[s[r + 1] - 1] if s[r + 1] > 0 else 0
        assert abs((b - a) - tot / P) <= u.max() + 1


def test_partition_edge_cases():
    assert sg.partition_rows(np.zeros(0, dtype=np.int64), 4).tolist() == [0, 0, 0, 0, 0]
    assert sg.partition_rows(np.zeros(5, dtype=np.int64), 2).tolist() == [0, 0, 5]
