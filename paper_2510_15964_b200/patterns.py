"""Atomic block-pattern pool (sf/patterns.py:24-133) + its device form.

The reference builds the pool offline (one sorted coordinate table per
pattern) and combines per-head assignments online. Here the same pool is
also lowered once to the two device forms the kernels consume:

* ``kinds/params`` (int32) — analytic membership used by the predictor's
  coverage selection kernel (csrc/mask_build.cu);
* attention tile tables (csrc/attn.cu) — per pattern, CSR over 64-row query
  tiles and CSC over 64-key tiles with 16x16-cell masks.

Pattern ids, order (the tie-break), coordinates and errors match the
reference exactly (pinned by tests/test_oracle_golden.py::test_pools_match_reference against tests/golden/pools.npz).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from .errors import PatternError

Coord = tuple[int, int]

KIND_CODES = {"blockdiag": 0, "band": 1, "causal": 2, "global": 3, "strided": 4, "dense": 5}


@dataclass(frozen=True)
class LayoutTable:
    """Precomputed active-block coordinates for one pattern (sf/patterns.py:24-45)."""

    pattern_id: str
    n_b: int
    coords: tuple[Coord, ...]
    kind: str = "dense"
    param: int = 0

    @property
    def active_blocks(self) -> int:
        return len(self.coords)

    def __post_init__(self):
        seen = set()
        for br, bc in self.coords:
            if not (0 <= br < self.n_b and 0 <= bc < self.n_b):
                raise PatternError(f"{self.pattern_id}: block ({br},{bc}) outside {self.n_b}x{self.n_b} grid")
            if (br, bc) in seen:
                raise PatternError(f"{self.pattern_id}: duplicate block ({br},{bc})")
            seen.add((br, bc))
        if tuple(sorted(self.coords)) != self.coords:
            raise PatternError(f"{self.pattern_id}: coordinates not sorted")


@dataclass(frozen=True)
class CombinedLayout:
    """Per-head layouts concatenated into one flat (head, br, bc) list (sf/patterns.py:48-60)."""

    n_b: int
    n_heads: int
    entries: tuple[tuple[int, int, int], ...]
    head_offsets: tuple[int, ...]

    def head_coords(self, head: int) -> tuple[Coord, ...]:
        lo = self.head_offsets[head]
        hi = self.head_offsets[head + 1] if head + 1 < self.n_heads else len(self.entries)
        return tuple((br, bc) for _, br, bc in self.entries[lo:hi])


def _member(kind: str, p: int, i: np.ndarray, j: np.ndarray) -> np.ndarray:
    d = i - j
    if kind == "blockdiag":
        return d == 0
    if kind == "band":
        return np.abs(d) <= p
    if kind == "causal":
        return (d >= 0) & (d <= p)
    if kind == "global":
        return (i < p) | (j < p) | (d == 0)
    if kind == "strided":
        return d % p == 0
    return np.ones_like(d, dtype=bool)


def _table(pid: str, kind: str, p: int, n_b: int) -> LayoutTable:
    i, j = np.meshgrid(np.arange(n_b), np.arange(n_b), indexing="ij")
    br, bc = np.nonzero(_member(kind, p, i, j))  # row-major = sorted
    return LayoutTable(pid, n_b, tuple(zip(br.tolist(), bc.tolist())), kind, p)


def build_pool(n_b: int, band_widths=(1, 2), global_sizes=(1,), strides=(2,), causal_widths=(1,)) -> dict[str, LayoutTable]:
    """Offline pool construction in the reference's fixed order (sf/patterns.py:88-120):
    blockdiag, band{w}..., causal{w}..., global{g}..., strided{p}..., dense."""
    if n_b < 1:
        raise PatternError(f"grid side must be >= 1, got {n_b}")
    specs = [("blockdiag", "blockdiag", 0)]
    for w in band_widths:
        if w > n_b:
            raise PatternError(f"band width {w} exceeds grid side {n_b}")
        specs.append((f"band{w}", "band", w))
    for w in causal_widths:
        if w > n_b:
            raise PatternError(f"causal width {w} exceeds grid side {n_b}")
        specs.append((f"causal{w}", "causal", w))
    for g in global_sizes:
        if g > n_b:
            raise PatternError(f"global border {g} exceeds grid side {n_b}")
        specs.append((f"global{g}", "global", g))
    for p in strides:
        if p > n_b:
            raise PatternError(f"stride {p} exceeds grid side {n_b}")
        specs.append((f"strided{p}", "strided", p))
    specs.append(("dense", "dense", 0))
    pool: dict[str, LayoutTable] = {}
    for pid, kind, p in specs:
        if pid not in pool:
            pool[pid] = _table(pid, kind, p, n_b)
    return pool


def combine_layouts(assignment: list[str], pool: dict[str, LayoutTable]) -> CombinedLayout:
    """Online pattern combination (sf/patterns.py:123-133)."""
    entries: list[tuple[int, int, int]] = []
    offsets: list[int] = []
    n_b = next(iter(pool.values())).n_b
    for head, pid in enumerate(assignment):
        if pid not in pool:
            raise PatternError(f"pattern id {pid!r} not in pool")
        offsets.append(len(entries))
        entries.extend((head, br, bc) for br, bc in pool[pid].coords)
    return CombinedLayout(n_b=n_b, n_heads=len(assignment), entries=tuple(entries), head_offsets=tuple(offsets))


# ---------------------------------------------------------------------------
# device lowering


@dataclass
class DevicePool:
    """The pool as the sm_100a kernels see it (built once per (pool, s, attn_blk, device))."""

    ids: list[str]
    kinds: object  # torch int32 [P]
    params: object  # torch int32 [P]
    tables: object | None  # torch int32 attention tile tables, 64x64 tiles (None until built for a seq_len)
    seq_len: int = 0
    attn_blk: int = 0
    index: dict = field(default_factory=dict)
    tables128: object | None = None  # 128x128-tile tables for the tcgen05 attention kernels

    def idx(self, pid: str) -> int:
        if pid not in self.index:
            raise PatternError(f"pattern id {pid!r} not in pool")
        return self.index[pid]


TILE = 64  # attention kernel tile edge (csrc/attn.cu kT)


def tables_from_grids(grids: np.ndarray, seq_len: int, attn_blk: int) -> np.ndarray:
    """Attention tile tables (csrc/attn.cu layout) for arbitrary block layouts: grids bool
    [P, n_b, n_b] -> int32 array. Same format the C-ABI builds for pool kinds."""
    from .errors import LayoutError, UnsupportedError

    if attn_blk % 16 or attn_blk < 16:
        raise UnsupportedError(f"attn_blk {attn_blk} unsupported on the sm_100a path (multiple of 16)")
    if seq_len % attn_blk:
        raise LayoutError(f"sequence length {seq_len} != n_b*blk")
    P = grids.shape[0]
    nt = -(-seq_len // TILE)
    per = 2 * (nt + 1) + 4 * nt * nt
    out = np.zeros(4 + P * per, np.int32)
    out[:4] = (nt, P, seq_len, attn_blk)
    nc = seq_len // 16
    ci = np.arange(nc)
    for p in range(P):
        cells = grids[p][np.ix_(ci * 16 // attn_blk, ci * 16 // attn_blk)]  # [nc, nc] active 16x16 cells
        tm = np.zeros((nt, nt), np.int64)
        for a in range(nc):
            for b in np.flatnonzero(cells[a]):
                tm[a // 4, b // 4] |= 1 << ((a % 4) * 4 + b % 4)
        base = 4 + p * per
        row_ptr, csr_col, csr_mask = base, base + nt + 1, base + nt + 1 + nt * nt
        col_ptr = csr_mask + nt * nt
        csc_row, csc_mask = col_ptr + nt + 1, col_ptr + nt + 1 + nt * nt
        n = 0
        for i in range(nt):
            out[row_ptr + i] = n
            for j in np.flatnonzero(tm[i]):
                out[csr_col + n], out[csr_mask + n] = j, tm[i, j]
                n += 1
        out[row_ptr + nt] = n
        n = 0
        for j in range(nt):
            out[col_ptr + j] = n
            for i in np.flatnonzero(tm[:, j]):
                out[csc_row + n], out[csc_mask + n] = i, tm[i, j]
                n += 1
        out[col_ptr + nt] = n
        if np.any(out[row_ptr + 1 : row_ptr + nt + 1] == out[row_ptr : row_ptr + nt]):
            raise LayoutError("a block-row has no active blocks (pattern pool violation)")
    return out


def tables128_from_grids(grids: np.ndarray, seq_len: int, attn_blk: int) -> np.ndarray:
    """128x128-tile tables for the tcgen05 attention kernels (csrc/attn_sm100.cu): per pattern
    row_ptr, csr_col, csr_lo, csr_hi, col_ptr, csc_row, csc_lo, csc_hi; a tile's 64-bit mask has
    bit (ci*8 + cj) set when its 16x16 cell (ci, cj) is active."""
    from .errors import LayoutError, UnsupportedError

    if attn_blk % 16 or attn_blk < 16:
        raise UnsupportedError(f"attn_blk {attn_blk} unsupported on the sm_100a path (multiple of 16)")
    if seq_len % attn_blk:
        raise LayoutError(f"sequence length {seq_len} != n_b*blk")
    T = 128
    P = grids.shape[0]
    nt = -(-seq_len // T)
    per = 2 * (nt + 1) + 6 * nt * nt
    out = np.zeros(4 + P * per, np.int64)
    out[:4] = (nt, P, seq_len, attn_blk)
    nc = seq_len // 16
    ci = np.arange(nc)
    for p in range(P):
        cells = grids[p][np.ix_(ci * 16 // attn_blk, ci * 16 // attn_blk)]
        tm = np.zeros((nt, nt), np.uint64)
        a_idx, b_idx = np.nonzero(cells)
        for a, b in zip(a_idx, b_idx):
            tm[a // 8, b // 8] |= np.uint64(1) << np.uint64((a % 8) * 8 + b % 8)
        base = 4 + p * per
        rp, cc, clo, chi = base, base + nt + 1, base + nt + 1 + nt * nt, base + nt + 1 + 2 * nt * nt
        cp = base + nt + 1 + 3 * nt * nt
        cr, rlo, rhi = cp + nt + 1, cp + nt + 1 + nt * nt, cp + nt + 1 + 2 * nt * nt
        n = 0
        for i in range(nt):
            out[rp + i] = n
            for j in np.flatnonzero(tm[i]):
                out[cc + n], out[clo + n], out[chi + n] = j, int(tm[i, j]) & 0xFFFFFFFF, int(tm[i, j]) >> 32
                n += 1
        out[rp + nt] = n
        n = 0
        for j in range(nt):
            out[cp + j] = n
            for i in np.flatnonzero(tm[:, j]):
                out[cr + n], out[rlo + n], out[rhi + n] = i, int(tm[i, j]) & 0xFFFFFFFF, int(tm[i, j]) >> 32
                n += 1
        out[cp + nt] = n
        if np.any(out[rp + 1 : rp + nt + 1] == out[rp : rp + nt]):
            raise LayoutError("a block-row has no active blocks (pattern pool violation)")
    return out.astype(np.uint32).view(np.int32)


def pool_grids(pool: dict[str, LayoutTable]) -> np.ndarray:
    n_b = next(iter(pool.values())).n_b
    grids = np.zeros((len(pool), n_b, n_b), bool)
    for i, t in enumerate(pool.values()):
        c = np.asarray(t.coords, dtype=np.int64).reshape(-1, 2)
        grids[i, c[:, 0], c[:, 1]] = True
    return grids


def device_pool(pool: dict[str, LayoutTable], device, seq_len: int | None = None, attn_blk: int | None = None) -> DevicePool:
    import torch

    from . import _abi

    ids = list(pool)
    if ids[-1] != "dense":
        raise PatternError("pool must end with 'dense'")
    kinds = np.array([KIND_CODES[pool[p].kind] for p in ids], np.int32)
    params = np.array([max(pool[p].param, 1) if pool[p].kind in ("strided",) else pool[p].param for p in ids], np.int32)
    dp = DevicePool(ids, torch.from_numpy(kinds).to(device), torch.from_numpy(params).to(device), None,
                    index={p: i for i, p in enumerate(ids)})
    if seq_len is not None:
        n = ctypes.c_int(0)
        _abi.lib().lx_attn_tables_size(len(ids), seq_len, attn_blk, ctypes.byref(n))
        host = np.zeros(n.value, np.int32)
        _abi.call("lx_attn_tables", kinds.ctypes.data, params.ctypes.data, len(ids), seq_len, attn_blk, host.ctypes.data, n.value)
        dp.tables = torch.from_numpy(host).to(device)
        dp.tables128 = torch.from_numpy(tables128_from_grids(pool_grids(pool), seq_len, attn_blk)).to(device)
        dp.seq_len, dp.attn_blk = seq_len, attn_blk
    return dp
