"""Seeded synthetic input generators shared by the tests, the bench and the oracle checks.

This module holds NO arithmetic of the method (no products, no accumulation, no
binning): it only builds input matrices A and B in CSR form.  Every random quantity is
a counter-based hash (SplitMix64) of (seed, position), so a matrix depends only on its
recipe, never on call order or thread count (DESIGN.md §"Input recipe").

Workloads follow BASELINE.json's configs as concretised in SURVEY.md §8(d):

* ``stencil(kind, n)``            — 2D5 / 2D9 / 3D7 / 3D27 Poisson matrices ([P:395]);
                                    lexicographic order, x fastest; diagonal = number of
                                    stencil neighbours, off-diagonals -1 ("coef" values).
* ``rmat(scale, ef, abcd, seed)`` — R-MAT power-law graph (configs 3a/3b), vertex ids
                                    relabelled by a seeded permutation, duplicates merged.
* ``band(n, lo, hi)`` / ``uniform_rows(n, r, seed)`` — config 5 band(64) × uniform(64).
* ``aggregation_P(n, smoothed)``  — 2×2×2 geometric aggregation prolongator for the
                                    3D7 Galerkin product (config 4); smoothed variant is
                                    P_s = (I - 1/8 A) P_t written out per stencil row.
* ``transpose``                   — materialises R = Pᵀ (input preparation only).
* ``random_csr`` / ``forced_u_pair`` — small randomized matrices for parity tests.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED = 150405022  # base seed from the arXiv id

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


@dataclass
class Csr:
    shape: tuple            # (rows, cols)
    rp: np.ndarray          # int64 [rows+1]
    ci: np.ndarray          # int32 [nnz]
    val: np.ndarray         # float64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.ci.shape[0])

    def row_lengths(self) -> np.ndarray:
        return np.diff(self.rp)

    def to_dense(self) -> np.ndarray:
        d = np.zeros(self.shape, dtype=np.float64)
        rows = np.repeat(np.arange(self.shape[0]), np.diff(self.rp))
        d[rows, self.ci] = self.val
        return d

    def pattern_dense(self) -> np.ndarray:
        d = np.zeros(self.shape, dtype=bool)
        rows = np.repeat(np.arange(self.shape[0]), np.diff(self.rp))
        d[rows, self.ci] = True
        return d


# ----------------------------------------------------------------------------- RNG
def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def hash3(seed: int, a, b) -> np.ndarray:
    """Counter-based hash of (seed, a, b) → uint64."""
    a = np.asarray(a).astype(np.uint64)
    b = np.asarray(b).astype(np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ splitmix64(a))
        return splitmix64(h ^ (b * np.uint64(0xD6E8FEB86659FD93) & _M64))


def values(seed: int, rows: np.ndarray, cols: np.ndarray, mode: str) -> np.ndarray:
    """Value of entry (i, j) as a function of its position only.

    ``int``  : s·(1 + h mod 8)          ∈ ±[1, 8]   (exact arithmetic at small sizes)
    ``real`` : s·(1 + h53·2^-53)        ∈ ±[1, 2)
    ``one``  : 1.0
    ``dyadic``: s·(1 + (h mod 8)/8)     ∈ ±[1, 2)  (exact for short sums)
    """
    if mode == "one":
        return np.ones(rows.shape[0], dtype=np.float64)
    h = hash3(seed, rows, cols)
    s = np.where((h >> np.uint64(63)) == 1, -1.0, 1.0)
    if mode == "int":
        return s * (1.0 + (h & np.uint64(7)).astype(np.float64))
    if mode == "dyadic":
        return s * (1.0 + (h & np.uint64(7)).astype(np.float64) / 8.0)
    if mode == "real":
        return s * (1.0 + ((h >> np.uint64(10)) & np.uint64((1 << 53) - 1)).astype(np.float64) * 2.0 ** -53)
    raise ValueError("unknown value mode %r" % mode)


def _from_coo_sorted(rows: np.ndarray, cols: np.ndarray, shape) -> tuple:
    """CSR (rp, ci) from (row, col) pairs already sorted by (row, col), duplicate-free."""
    m = shape[0]
    counts = np.bincount(rows, minlength=m) if rows.size else np.zeros(m, dtype=np.int64)
    rp = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    return rp, cols.astype(np.int32)


def from_coo(rows, cols, shape, vals=None, dedup: bool = True) -> Csr:
    """Build a sorted CSR from unsorted COO; duplicates are merged (kept once)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    key = rows * np.int64(max(shape[1], 1)) + cols
    order = np.argsort(key, kind="stable")
    key = key[order]
    if dedup and key.size:
        keep = np.ones(key.size, dtype=bool)
        keep[1:] = key[1:] != key[:-1]
        order = order[keep]
        key = key[keep]
    r = rows[order]
    c = cols[order]
    rp, ci = _from_coo_sorted(r, c, shape)
    v = np.asarray(vals, dtype=np.float64)[order] if vals is not None else np.ones(ci.size)
    return Csr(tuple(shape), rp, ci, v)


def with_values(M: Csr, mode: str, seed: int) -> Csr:
    rows = np.repeat(np.arange(M.shape[0], dtype=np.int64), np.diff(M.rp))
    return Csr(M.shape, M.rp, M.ci, values(seed, rows, M.ci.astype(np.int64), mode))


# ------------------------------------------------------------------------ stencils
_STENCILS = {
    "2d5": (2, [(dx, dy) for dy in (-1, 0, 1) for dx in (-1, 0, 1) if abs(dx) + abs(dy) <= 1]),
    "2d9": (2, [(dx, dy) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]),
    "3d7": (3, [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)
                if abs(dx) + abs(dy) + abs(dz) <= 1]),
    "3d27": (3, [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]),
}


def stencil(kind: str, n: int, mode: str = "coef", seed: int = SEED + 3) -> Csr:
    """Poisson stencil matrix on an n^d grid (SPEC gen_poisson [S:53-61]).

    Offsets are visited in ascending linear order, so each row's columns come out
    sorted.  ``coef``: diagonal = (#stencil points - 1), neighbours -1.
    """
    dim, offs = _STENCILS[kind]
    N = n ** dim
    idx = np.arange(N, dtype=np.int64)
    x = idx % n
    y = (idx // n) % n
    z = idx // (n * n) if dim == 3 else np.zeros_like(idx)
    lin = sorted(offs, key=lambda o: (o[2] if dim == 3 else 0) * n * n + o[1] * n + o[0])
    K = len(lin)
    cols = np.full((N, K), -1, dtype=np.int64)
    for t, o in enumerate(lin):
        dx, dy = o[0], o[1]
        dz = o[2] if dim == 3 else 0
        ok = (x + dx >= 0) & (x + dx < n) & (y + dy >= 0) & (y + dy < n)
        if dim == 3:
            ok &= (z + dz >= 0) & (z + dz < n)
        cols[ok, t] = idx[ok] + dz * n * n + dy * n + dx
    valid = cols >= 0
    counts = valid.sum(axis=1)
    rp = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    ci = cols[valid].astype(np.int32)
    del cols
    if mode == "coef":
        rows = np.repeat(idx, counts)
        val = np.where(ci.astype(np.int64) == rows, float(K - 1), -1.0)
    else:
        rows = np.repeat(idx, counts)
        val = values(seed, rows, ci.astype(np.int64), mode)
    return Csr((N, N), rp, ci, val)


# ---------------------------------------------------------------------------- R-MAT
def permutation(seed: int, n: int) -> np.ndarray:
    """Seeded permutation of range(n): argsort of hashed keys."""
    return np.argsort(hash3(seed, np.arange(n, dtype=np.int64), 0), kind="stable").astype(np.int64)


def rmat(scale: int, ef: int = 16, abcd=(0.45, 0.15, 0.15, 0.25), seed: int = SEED,
         mode: str = "real", vseed: int = SEED + 3, chunk: int = 1 << 22) -> Csr:
    """R-MAT graph: per edge and level one uniform draw picks
    the quadrant (bits MSB-first); vertex ids relabelled by a seeded permutation;
    directed; duplicates merged; self-loops kept."""
    n = 1 << scale
    E = ef * n
    a, b, c, _ = abcd
    t1, t2, t3 = a, a + b, a + b + c
    perm = permutation(seed + 2, n)
    src = np.empty(E, dtype=np.int64)
    dst = np.empty(E, dtype=np.int64)
    for e0 in range(0, E, chunk):
        e = np.arange(e0, min(E, e0 + chunk), dtype=np.int64)
        r = np.zeros(e.size, dtype=np.int64)
        cc = np.zeros(e.size, dtype=np.int64)
        for lvl in range(scale):
            u = (hash3(seed, e, lvl) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
            bit = np.int64(1 << (scale - 1 - lvl))
            rb = u >= t2            # quadrants (1,0) and (1,1) set the row bit
            cb = ((u >= t1) & (u < t2)) | (u >= t3)
            r |= np.where(rb, bit, 0)
            cc |= np.where(cb, bit, 0)
        src[e0:e0 + e.size] = perm[r]
        dst[e0:e0 + e.size] = perm[cc]
    M = from_coo(src, dst, (n, n))
    return with_values(M, mode, vseed)


# ------------------------------------------------------------------ band × uniform
def band(n: int, lo: int = 32, hi: int = 31, mode: str = "real", seed: int = SEED + 3,
         rows: tuple | None = None) -> Csr:
    """Row i holds columns [i-lo, i+hi] ∩ [0, n) (config 5's A); ``rows`` restricts to a
    row block [r0, r1) of the full matrix (the block keeps global column ids)."""
    r0, r1 = (0, n) if rows is None else rows
    i = np.arange(r0, r1, dtype=np.int64)
    w = lo + hi + 1
    cols = i[:, None] + np.arange(-lo, hi + 1, dtype=np.int64)[None, :]
    ok = (cols >= 0) & (cols < n)
    counts = ok.sum(axis=1)
    rp = np.zeros(r1 - r0 + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    ci = cols[ok]
    rr = np.repeat(i, counts)
    return Csr((r1 - r0, n), rp, ci.astype(np.int32), values(seed, rr, ci, mode))


def uniform_rows(n_rows: int, n_cols: int, r: int = 64, seed: int = SEED + 1, mode: str = "real",
                 vseed: int = SEED + 4) -> Csr:
    """Each row holds r distinct uniform columns (counter hash keyed by (seed, row, t));
    rows with a collision redraw their duplicates from further counters; sorted."""
    rows = np.arange(n_rows, dtype=np.int64)
    t = np.arange(r, dtype=np.int64)
    cols = (hash3(seed, rows[:, None], t[None, :]) % np.uint64(n_cols)).astype(np.int64)
    cols.sort(axis=1)
    dup = np.zeros(cols.shape, dtype=bool)
    dup[:, 1:] = cols[:, 1:] == cols[:, :-1]
    bad = np.nonzero(dup.any(axis=1))[0]
    for i in bad:
        got = list(dict.fromkeys(cols[i].tolist()))
        tt = r
        while len(got) < r:
            cnew = int(hash3(seed, np.int64(i), np.int64(tt)) % np.uint64(n_cols))
            tt += 1
            if cnew not in got:
                got.append(cnew)
        cols[i] = np.sort(np.array(got, dtype=np.int64))
    rp = np.arange(n_rows + 1, dtype=np.int64) * r
    ci = cols.reshape(-1)
    return Csr((n_rows, n_cols), rp, ci.astype(np.int32),
               values(vseed, np.repeat(rows, r), ci, mode))


# -------------------------------------------------------------- Galerkin operators
def aggregation_P(n: int, smoothed: bool = False) -> Csr:
    """2×2×2 geometric aggregation prolongator for the 3D7 Laplacian on n^3 (n even).

    Tentative: P[i, agg(i)] = 1 with agg = ((z>>1)·(n/2) + (y>>1))·(n/2) + (x>>1).
    Smoothed (ω = 3/4, D = 6I ⇒ ωD⁻¹ = 1/8): P_s = (I - A/8)·P_t, written out per row:
    P_s[i, g] = [agg(i)=g]·(1 - 6/8) + (1/8)·#{stencil neighbours j of i with agg(j)=g}.
    Values are dyadic (5/8, 1/8), so every Galerkin sum is exact.
    """
    assert n % 2 == 0
    N = n ** 3
    h = n // 2
    idx = np.arange(N, dtype=np.int64)
    x, y, z = idx % n, (idx // n) % n, idx // (n * n)
    agg = ((z >> 1) * h + (y >> 1)) * h + (x >> 1)
    if not smoothed:
        return Csr((N, h ** 3), np.arange(N + 1, dtype=np.int64), agg.astype(np.int32), np.ones(N))
    offs = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
    # Each row: own aggregate + up to 3 distinct foreign aggregates (one per axis).
    gcols = [agg]
    gvals = [np.full(N, 1.0 - 6.0 / 8.0)]
    for dx, dy, dz in offs:
        ok = (x + dx >= 0) & (x + dx < n) & (y + dy >= 0) & (y + dy < n) & (z + dz >= 0) & (z + dz < n)
        j = idx + dz * n * n + dy * n + dx
        gj = np.where(ok, agg[np.where(ok, j, 0)], -1)
        gcols.append(gj)
        gvals.append(np.where(ok, 1.0 / 8.0, 0.0))
    G = np.stack(gcols, axis=1)
    V = np.stack(gvals, axis=1)
    # merge equal aggregate ids within each row (sum of 1/8 contributions)
    order = np.argsort(np.where(G < 0, np.iinfo(np.int64).max, G), axis=1, kind="stable")
    G = np.take_along_axis(G, order, axis=1)
    V = np.take_along_axis(V, order, axis=1)
    K = G.shape[1]
    out_c = np.full((N, K), -1, dtype=np.int64)
    out_v = np.zeros((N, K))
    pos = np.zeros(N, dtype=np.int64)
    prev = np.full(N, -2, dtype=np.int64)
    for t in range(K):
        g, v = G[:, t], V[:, t]
        valid = g >= 0
        new = valid & (g != prev)
        same = valid & (g == prev)
        out_v[same, pos[same] - 1] += v[same]
        out_c[new, pos[new]] = g[new]
        out_v[new, pos[new]] = v[new]
        pos = pos + new
        prev = np.where(valid, g, prev)
    valid = out_c >= 0
    rp = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(valid.sum(axis=1), out=rp[1:])
    return Csr((N, h ** 3), rp, out_c[valid].astype(np.int32), out_v[valid])


def _to_scipy(M: Csr):
    import scipy.sparse as sp
    return sp.csr_matrix((M.val, M.ci.astype(np.int64), M.rp), shape=M.shape)


def _from_scipy(S) -> Csr:
    S = S.tocsr()
    S.sum_duplicates()
    S.sort_indices()
    return Csr(S.shape, S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data.astype(np.float64))


def amg_levels(kind: str, n: int, levels: int = 3, omega: float = 0.75):
    """The paper's Galerkin workload ([P:393-397]): an AMG hierarchy of a Poisson problem with
    smoothed aggregation and a Jacobi smoother.  Level 0: A = stencil(kind, n) (2D 5/9-point
    on n², 3D 7/27-point on n³).  Each level aggregates 2 (2D: 2×2, 3D: 2×2×2) neighbouring
    grid points of the level's grid (ceil(n/2) points per axis; odd n leaves boundary
    aggregates of one point), P_t[i, agg(i)] = 1, P = (I − ω D⁻¹ A)·P_t (Jacobi smoothing,
    ω = 3/4: reading Q15), R = Pᵀ, and the next level's operator is A' = R·A·P.
    Returns [(A_l, P_l, R_l)] for l < levels.  Input construction only (scipy.sparse); the
    products the benchmark and tests run on these inputs go through libspgemm / the oracle.
    Stored zeros from exact cancellation are dropped by scipy (any valid CSR is an input)."""
    import scipy.sparse as sp
    dim = _STENCILS[kind][0]
    A = _to_scipy(stencil(kind, n))
    out = []
    g = n
    for _ in range(levels):
        h = (g + 1) // 2
        N = g ** dim
        idx = np.arange(N, dtype=np.int64)
        x, y = idx % g, (idx // g) % g
        if dim == 2:
            agg = (y >> 1) * h + (x >> 1)
        else:
            z = idx // (g * g)
            agg = ((z >> 1) * h + (y >> 1)) * h + (x >> 1)
        Pt = sp.csr_matrix((np.ones(N), agg, np.arange(N + 1)), shape=(N, h ** dim))
        Dinv = sp.diags(1.0 / A.diagonal())
        P = (Pt - omega * (Dinv @ (A @ Pt))).tocsr()
        R = P.T.tocsr()
        out.append((_from_scipy(A), _from_scipy(P), _from_scipy(R)))
        A = (R @ (A @ P)).tocsr()
        g = h
    return out


def transpose(M: Csr) -> Csr:
    """Rᵀ materialisation (stable: rows of the transpose keep ascending columns)."""
    m, n = M.shape
    rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(M.rp))
    order = np.argsort(M.ci, kind="stable")
    tr = M.ci[order].astype(np.int64)
    tc = rows[order]
    rp, ci = _from_coo_sorted(tr, tc, (n, m))
    return Csr((n, m), rp, ci, M.val[order].copy())


# ------------------------------------------------------------------ small randoms
def random_csr(m: int, n: int, density: float, seed: int, mode: str = "int",
               zero_frac: float = 0.0) -> Csr:
    """Bernoulli(density) pattern; values by ``mode``; a fraction of stored entries set
    to explicit 0.0 (structural zeros stay in the pattern, [P:169])."""
    i = np.arange(m, dtype=np.int64)[:, None]
    j = np.arange(n, dtype=np.int64)[None, :]
    u = (hash3(seed, i, j) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    mask = u < density
    rows, cols = np.nonzero(mask)
    M = from_coo(rows, cols, (m, n))
    M = with_values(M, mode, seed + 1)
    if zero_frac > 0 and M.nnz:
        z = (hash3(seed + 2, np.arange(M.nnz), 7) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        M.val[z < zero_frac] = 0.0
    return M


def random_rows(m: int, n: int, lengths: np.ndarray, seed: int, mode: str = "int") -> Csr:
    """Row i holds lengths[i] distinct uniform columns in [0, n) (sorted)."""
    lengths = np.minimum(np.asarray(lengths, dtype=np.int64), n)
    rows_l, cols_l = [], []
    for i in range(m):
        L = int(lengths[i])
        if L == 0:
            continue
        if L * 4 >= n:
            u = hash3(seed, np.int64(i), np.arange(n, dtype=np.int64))
            c = np.sort(np.argsort(u, kind="stable")[:L])
        else:
            got = []
            seen = set()
            t = 0
            while len(got) < L:
                cc = int(hash3(seed, np.int64(i), np.int64(t)) % np.uint64(n))
                t += 1
                if cc not in seen:
                    seen.add(cc)
                    got.append(cc)
            c = np.sort(np.array(got, dtype=np.int64))
        rows_l.append(np.full(L, i, dtype=np.int64))
        cols_l.append(c)
    rows = np.concatenate(rows_l) if rows_l else np.zeros(0, dtype=np.int64)
    cols = np.concatenate(cols_l) if cols_l else np.zeros(0, dtype=np.int64)
    rp, ci = _from_coo_sorted(rows, cols, (m, n))
    return with_values(Csr((m, n), rp, ci, np.ones(ci.size)), mode, seed + 1)


def forced_u_pair(us, n: int, seed: int, mode: str = "int", dup: float = 0.0):
    """(A, B) with prescribed upper bounds: row i of A·B has exactly u_i = us[i]
    intermediate products (stage-1 bound [P:198-212]).  Row i of A picks a set of B
    rows whose lengths sum to us[i]; ``dup`` ∈ [0,1) makes B rows overlap (columns
    drawn from a window of size ~ u·(1-dup)) so nnz(c_i) < u_i."""
    us = [int(u) for u in us]
    b_lengths = []
    a_rows = []
    for i, u in enumerate(us):
        parts = []
        rem = u
        t = 0
        while rem > 0:
            h = int(hash3(seed, np.int64(i), np.int64(1000 + t)) % np.uint64(64)) + 1
            L = min(rem, h, n)
            parts.append(L)
            rem -= L
            t += 1
        ids = []
        for L in parts:
            ids.append(len(b_lengths))
            b_lengths.append(L)
        a_rows.append(ids)
    k = max(len(b_lengths), 1)
    # B rows: columns drawn inside a per-A-row window to control duplication
    b_rows, b_cols = [], []
    for i, ids in enumerate(a_rows):
        u = us[i]
        win = min(n, max(64, int(round(u * (1.0 - dup))))) if dup > 0 else n
        base = int(hash3(seed + 7, np.int64(i), 0) % np.uint64(max(n - win + 1, 1)))
        for bj in ids:
            L = b_lengths[bj]
            L = min(L, win)
            u_ = hash3(seed + 9, np.int64(bj), np.arange(win, dtype=np.int64))
            c = np.sort(np.argsort(u_, kind="stable")[:L]) + base
            b_rows.append(np.full(L, bj, dtype=np.int64))
            b_cols.append(c)
    br = np.concatenate(b_rows) if b_rows else np.zeros(0, dtype=np.int64)
    bc = np.concatenate(b_cols) if b_cols else np.zeros(0, dtype=np.int64)
    B = from_coo(br, bc, (k, n))
    B = with_values(B, mode, seed + 11)
    ar, ac = [], []
    for i, ids in enumerate(a_rows):
        for bj in ids:
            ar.append(i)
            ac.append(bj)
    A = from_coo(np.array(ar, dtype=np.int64), np.array(ac, dtype=np.int64), (len(us), k))
    A = with_values(A, mode, seed + 13)
    return A, B
