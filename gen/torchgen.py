"""Torch versions of the large generators of gen/ (bit-identical output, any device).

Used by bench.py to build the full-size configs on the GPU in seconds; tests/test_gen.py
checks every function against its numpy twin in gen/__init__.py on CPU tensors.  Like gen/,
this module holds no arithmetic of the method: only seeded input construction.

int64 arithmetic wraps mod 2^64 in torch, so SplitMix64 is exact; logical right shifts are an
arithmetic shift followed by a mask.
"""
from __future__ import annotations

import torch

from . import SEED, Csr

_K1 = -7046029254386353131    # 0x9E3779B97F4A7C15 as int64
_K2 = -4658895280553007687    # 0xBF58476D1CE4E5B9
_K3 = -7723592293110705685    # 0x94D049BB133111EB
_K4 = -2960836687051489901    # 0xD6E8FEB86659FD93


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    z = x + _K1
    z = (z ^ _srl(z, 30)) * _K2
    z = (z ^ _srl(z, 27)) * _K3
    return z ^ _srl(z, 31)


def _as_i64(v: int) -> int:
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def hash3(seed: int, a: torch.Tensor, b) -> torch.Tensor:
    """Same as gen.hash3 (returns int64 holding the uint64 bit pattern)."""
    a = torch.as_tensor(a, dtype=torch.int64)
    b = torch.as_tensor(b, dtype=torch.int64, device=a.device)
    h = splitmix64(torch.full((), _as_i64(seed), dtype=torch.int64, device=a.device) ^ splitmix64(a))
    return splitmix64(h ^ (b * _K4))


def _u53(h: torch.Tensor) -> torch.Tensor:
    """(h >> 11) as float64 in [0, 2^53)."""
    return _srl(h, 11).to(torch.float64)


def values(seed: int, rows: torch.Tensor, cols: torch.Tensor, mode: str) -> torch.Tensor:
    if mode == "one":
        return torch.ones(rows.shape[0], dtype=torch.float64, device=rows.device)
    h = hash3(seed, rows, cols)
    s = torch.where(_srl(h, 63) == 1, -1.0, 1.0).to(torch.float64)
    if mode == "int":
        return s * (1.0 + (h & 7).to(torch.float64))
    if mode == "dyadic":
        return s * (1.0 + (h & 7).to(torch.float64) / 8.0)
    if mode == "real":
        return s * (1.0 + (_srl(h, 10) & ((1 << 53) - 1)).to(torch.float64) * 2.0 ** -53)
    raise ValueError(mode)


def band(n: int, lo: int = 32, hi: int = 31, mode: str = "real", seed: int = SEED + 3, rows=None,
         device="cuda"):
    """gen.band on `device`: returns (rp, ci, val) tensors and the shape."""
    r0, r1 = (0, n) if rows is None else rows
    i = torch.arange(r0, r1, dtype=torch.int64, device=device)
    cols = i[:, None] + torch.arange(-lo, hi + 1, dtype=torch.int64, device=device)[None, :]
    ok = (cols >= 0) & (cols < n)
    counts = ok.sum(dim=1)
    rp = torch.zeros(r1 - r0 + 1, dtype=torch.int64, device=device)
    rp[1:] = torch.cumsum(counts, 0)
    ci = cols[ok]
    rr = torch.repeat_interleave(i, counts)
    return (rp, ci.to(torch.int32), values(seed, rr, ci, mode)), (r1 - r0, n)


def uniform_rows(n_rows: int, n_cols: int, r: int = 64, seed: int = SEED + 1, mode: str = "real",
                 vseed: int = SEED + 4, device="cuda", chunk: int = 1 << 20, first_row: int = 0):
    """gen.uniform_rows on `device` (rows with a collision redraw from further counters).
    first_row > 0: rows [first_row, first_row + n_rows) of the same matrix (a rank's slice)."""
    rp = torch.arange(n_rows + 1, dtype=torch.int64, device=device) * r
    ci = torch.empty(n_rows * r, dtype=torch.int32, device=device)
    val = torch.empty(n_rows * r, dtype=torch.float64, device=device)
    t = torch.arange(r, dtype=torch.int64, device=device)
    for r0 in range(0, n_rows, chunk):
        r1 = min(n_rows, r0 + chunk)
        rows = torch.arange(first_row + r0, first_row + r1, dtype=torch.int64, device=device)
        h = hash3(seed, rows[:, None], t[None, :])
        cols = _srl(h, 0)  # bit pattern
        # uint64 modulo n_cols: split into high/low 32-bit halves (exact in int64)
        hi_ = _srl(cols, 32)
        lo_ = cols & 0xFFFFFFFF
        cols = (((hi_ % n_cols) * ((1 << 32) % n_cols)) % n_cols + lo_ % n_cols) % n_cols
        cols, _ = torch.sort(cols, dim=1)
        dup = torch.zeros_like(cols, dtype=torch.bool)
        dup[:, 1:] = cols[:, 1:] == cols[:, :-1]
        bad = torch.nonzero(dup.any(dim=1)).flatten().tolist()
        if bad:
            cols_cpu = cols.cpu()
            for b in bad:
                i = first_row + r0 + b
                got = list(dict.fromkeys(cols_cpu[b].tolist()))
                tt = r
                while len(got) < r:
                    hv = int(hash3(seed, torch.tensor(i), torch.tensor(tt)).item()) & ((1 << 64) - 1)
                    cnew = hv % n_cols
                    tt += 1
                    if cnew not in got:
                        got.append(cnew)
                cols_cpu[b] = torch.tensor(sorted(got), dtype=torch.int64)
            cols = cols_cpu.to(device)
        ci[r0 * r:r1 * r] = cols.reshape(-1).to(torch.int32)
        val[r0 * r:r1 * r] = values(vseed, torch.repeat_interleave(rows, r), cols.reshape(-1), mode)
    return (rp, ci, val), (n_rows, n_cols)


def rmat(scale: int, ef: int = 16, abcd=(0.45, 0.15, 0.15, 0.25), seed: int = SEED, mode: str = "real",
         vseed: int = SEED + 3, device="cuda", chunk: int = 1 << 24):
    """gen.rmat on `device`: same per-edge draws, permutation, dedup and values."""
    n = 1 << scale
    E = ef * n
    a, b, c, _ = abcd
    t1, t2, t3 = a, a + b, a + b + c
    # permutation: argsort of hashed keys (stable) — uint64 order via signed order of x ^ 2^63
    keys = hash3(seed + 2, torch.arange(n, dtype=torch.int64, device=device), 0) ^ (-(1 << 63))
    perm = torch.sort(keys, stable=True).indices
    src = torch.empty(E, dtype=torch.int64, device=device)
    dst = torch.empty(E, dtype=torch.int64, device=device)
    for e0 in range(0, E, chunk):
        e = torch.arange(e0, min(E, e0 + chunk), dtype=torch.int64, device=device)
        r = torch.zeros_like(e)
        cc = torch.zeros_like(e)
        for lvl in range(scale):
            u = _u53(hash3(seed, e, lvl)) * 2.0 ** -53
            bit = 1 << (scale - 1 - lvl)
            rb = u >= t2
            cb = ((u >= t1) & (u < t2)) | (u >= t3)
            r |= rb.to(torch.int64) * bit
            cc |= cb.to(torch.int64) * bit
        src[e0:e0 + e.numel()] = perm[r]
        dst[e0:e0 + e.numel()] = perm[cc]
    key = torch.unique(src * n + dst)  # sorted, duplicates merged
    rows, cols = key // n, key % n
    counts = torch.bincount(rows, minlength=n)
    rp = torch.zeros(n + 1, dtype=torch.int64, device=device)
    rp[1:] = torch.cumsum(counts, 0)
    return (rp, cols.to(torch.int32), values(vseed, rows, cols, mode)), (n, n)


def to_csr(t, shape) -> Csr:
    rp, ci, val = t
    return Csr(tuple(shape), rp.cpu().numpy(), ci.cpu().numpy(), val.cpu().numpy())
