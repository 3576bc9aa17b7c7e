"""Atomic block-pattern pool (sf/patterns.py:24-133) + its device form.

The reference builds the pool offline (one sorted coordinate table per
pattern) and combines per-head assignments online. Here the same pool is
also lowered once to the two device forms the kernels consume:

* ``kinds/params`` (int32) — analytic membership used by the predictor's
  coverage selection kernel (csrc/mask_build.cu);
* gathered 128-tile attention tables (csrc/attn_sm100.cu, tables128_from_grids)
  — per pattern, CSR over 128-query tiles and CSC over 128-key tiles whose
  entries stack the active gather units (gcd(attn_blk, 128) tokens) with
  64-bit masks of active 16x16 cells.

Pattern ids, order (the tie-break), coordinates and errors match the
reference exactly (pinned by tests/test_oracle_golden.py::test_pools_match_reference against tests/golden/pools.npz).
"""

from __future__ import annotations

import math
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
    tables: object | None  # torch int32 gathered 128-tile attention tables (tables128_from_grids), None until built
    seq_len: int = 0
    attn_blk: int = 0
    index: dict = field(default_factory=dict)

    @property
    def tables128(self):
        return self.tables

    @property
    def gather_rows(self) -> int:
        """Rows per gather unit of the attention tables: gcd(attn_blk, 128)."""
        return math.gcd(self.attn_blk, 128)

    def idx(self, pid: str) -> int:
        if pid not in self.index:
            raise PatternError(f"pattern id {pid!r} not in pool")
        return self.index[pid]


GATHER_SLOTS = 8  # unit slots per gathered 128-row tile (128 / 16)
ENTRY_INTS = 2 + GATHER_SLOTS  # lo, hi, unit ids


def tables128_from_grids(grids: np.ndarray, seq_len: int, attn_blk: int) -> np.ndarray:
    """Gathered 128x128-tile tables for the tcgen05 attention kernels (csrc/attn_sm100.cu), so the work of a
    tile list is proportional to the active blocks, not to the 128-tiles they touch.

    A gather unit is gu = min(attn_blk, 128) consecutive tokens (one block, or a 128-token tile of a larger
    block); a gathered tile is nsub = 128 / gu units stacked, loaded as nsub TMA boxes of gu rows.
      CSR (forward, dQ): for query tile i (128 contiguous queries) the ascending union of the key units any
        of its rows attends to, packed nsub per entry;
      CSC (dK/dV): for key tile j (128 contiguous keys) the ascending union of the query units attending
        to it, packed nsub per entry.
    An entry is [lo, hi, u_0 .. u_7]: the 64-bit mask (bit a*8 + b) of active 16x16 cells, a the query cell
    and b the key cell inside the (gathered) tile, and the unit ids of its slots. Unused slots repeat the
    entry's first unit with no mask bit set (real, finite data; contributes nothing).

    int32 layout: header [nt, P, seq_len, attn_blk, gu, nsub, per, 0]; per pattern p at 8 + p * per:
    row_ptr[nt + 1], col_ptr[nt + 1], csr[nt * nt][10], csc[nt * nt][10]."""
    from .errors import LayoutError, UnsupportedError

    if attn_blk % 16 or attn_blk < 16:
        raise UnsupportedError(f"attn_blk {attn_blk} unsupported on the sm_100a path (multiple of 16)")
    if seq_len % attn_blk:
        raise LayoutError(f"sequence length {seq_len} != n_b*blk")
    T = 128
    gu = math.gcd(attn_blk, T)  # largest power of two <= 128 dividing the block
    nsub = T // gu
    cpu = gu // 16  # 16-cells per unit
    P = grids.shape[0]
    nt = -(-seq_len // T)
    n_units = seq_len // gu
    per = 2 * (nt + 1) + 2 * ENTRY_INTS * nt * nt
    out = np.zeros(8 + P * per, np.int64)
    out[:8] = (nt, P, seq_len, attn_blk, gu, nsub, per, 0)
    nc = seq_len // 16
    ci = np.arange(nc)
    for p in range(P):
        cells = grids[p][np.ix_(ci * 16 // attn_blk, ci * 16 // attn_blk)]  # [nc, nc] active 16x16 cells
        cells_pad = np.zeros((nt * 8, nt * 8), bool)
        cells_pad[:nc, :nc] = cells
        base = 8 + p * per
        rp, cp = base, base + nt + 1
        csr0, csc0 = cp + nt + 1, cp + nt + 1 + ENTRY_INTS * nt * nt
        if np.any(~cells.any(1)):
            raise LayoutError("a block-row has no active blocks (pattern pool violation)")
        for transpose, ptr, ent0 in ((False, rp, csr0), (True, cp, csc0)):
            cm = cells_pad.T if transpose else cells_pad  # rows: the tile side, cols: the gathered side
            n = 0
            for t in range(nt):
                out[ptr + t] = n
                rows = cm[t * 8 : (t + 1) * 8]  # [8 cells of the tile, nt*8 cells]
                unit_act = rows[:, : n_units * cpu].reshape(8, n_units, cpu).any(axis=(0, 2))
                units = np.flatnonzero(unit_act)
                for c0 in range(0, len(units), nsub):
                    grp = units[c0 : c0 + nsub]
                    mask = 0
                    for slot, u in enumerate(grp):
                        sub = rows[:, u * cpu : (u + 1) * cpu]  # [8, cpu]
                        for a, b in zip(*np.nonzero(sub)):
                            qa, kb = (slot * cpu + b, a) if transpose else (a, slot * cpu + b)
                            mask |= 1 << (qa * 8 + kb)
                    e = ent0 + n * ENTRY_INTS
                    out[e], out[e + 1] = mask & 0xFFFFFFFF, mask >> 32
                    out[e + 2 : e + 2 + nsub] = np.concatenate([grp, np.full(nsub - len(grp), grp[0])])
                    n += 1
            out[ptr + nt] = n
    return out.astype(np.uint32).view(np.int32)


def tables128_work(tables: np.ndarray, p: int = 0) -> tuple[int, int]:
    """(forward / dQ gathered tiles, dK/dV gathered tiles) of pattern p: the kernels' work units."""
    t = np.asarray(tables).view(np.int32)
    nt, per = int(t[0]), int(t[6])
    base = 8 + p * per
    return int(t[base + nt]), int(t[base + nt + 1 + nt])


def pool_grids(pool: dict[str, LayoutTable]) -> np.ndarray:
    n_b = next(iter(pool.values())).n_b
    grids = np.zeros((len(pool), n_b, n_b), bool)
    for i, t in enumerate(pool.values()):
        c = np.asarray(t.coords, dtype=np.int64).reshape(-1, 2)
        grids[i, c[:, 0], c[:, 1]] = True
    return grids


def device_pool(pool: dict[str, LayoutTable], device, seq_len: int | None = None, attn_blk: int | None = None) -> DevicePool:
    import torch

    ids = list(pool)
    if ids[-1] != "dense":
        raise PatternError("pool must end with 'dense'")
    kinds = np.array([KIND_CODES[pool[p].kind] for p in ids], np.int32)
    params = np.array([max(pool[p].param, 1) if pool[p].kind in ("strided",) else pool[p].param for p in ids], np.int32)
    dp = DevicePool(ids, torch.from_numpy(kinds).to(device), torch.from_numpy(params).to(device), None,
                    index={p: i for i, p in enumerate(ids)})
    if seq_len is not None:
        dp.tables = torch.from_numpy(tables128_from_grids(pool_grids(pool), seq_len, attn_blk)).to(device)
        dp.seq_len, dp.attn_blk = seq_len, attn_blk
    return dp
