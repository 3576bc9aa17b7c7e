"""Gathered 128-tile attention tables (patterns.tables128_from_grids): host logic, CPU only.

The CSR side (forward, dQ) and the CSC side (dK/dV) must each reproduce exactly the active 16x16
cells of the layout (sf/block_sparse.py semantics: a block is computed iff it is in the layout), every
entry's units ascending and unique except for the padding that repeats the first unit with no mask bit,
and the work (entries) must equal the ceil(|union of units| / nsub) per tile."""

import numpy as np
import pytest

from oracle import sf_oracle as O
from paper_2510_15964_b200 import patterns as PT


def decode(tab, p, seq_len):
    t = np.asarray(tab).view(np.int32)
    nt, P, s, ab, gu, nsub, per = (int(x) for x in t[:7])
    base = 8 + p * per
    rp, cp = base, base + nt + 1
    csr0, csc0 = cp + nt + 1, cp + nt + 1 + PT.ENTRY_INTS * nt * nt
    nc = seq_len // 16
    cpu = gu // 16
    out = []
    for transpose, ptr, ent0 in ((False, rp, csr0), (True, cp, csc0)):
        cells = np.zeros((nt * 8, nt * 8), bool)
        for tile in range(nt):
            for e in range(t[ptr + tile], t[ptr + tile + 1]):
                ent = t[ent0 + e * PT.ENTRY_INTS : ent0 + (e + 1) * PT.ENTRY_INTS]
                mask = (int(np.uint32(ent[0])) | (int(np.uint32(ent[1])) << 32))
                units = [int(u) for u in ent[2 : 2 + nsub]]
                used = [u for k, u in enumerate(units) if any((mask >> ((k * cpu + b) * 8 + a if transpose else a * 8 + k * cpu + b)) & 1
                                                               for a in range(8) for b in range(cpu))]
                assert used == sorted(set(used))
                for bit in range(64):
                    if (mask >> bit) & 1:
                        a, b = divmod(bit, 8)  # a: query cell in the (gathered) tile, b: key cell
                        if transpose:
                            q = units[a // cpu] * cpu + a % cpu
                            k = tile * 8 + b
                        else:
                            q = tile * 8 + a
                            k = units[b // cpu] * cpu + b % cpu
                        assert not cells[q, k]
                        cells[q, k] = True
        out.append(cells[:nc, :nc])
    return out


def grid_cells(grid, seq_len, ab):
    ci = np.arange(seq_len // 16)
    return grid[np.ix_(ci * 16 // ab, ci * 16 // ab)]


@pytest.mark.parametrize("s,ab", [(64, 16), (128, 32), (192, 64), (512, 64), (512, 16), (1024, 128), (2048, 256), (256, 128)])
def test_gathered_tables_cover_layout_exactly(s, ab):
    n_b = s // ab
    rng = np.random.default_rng(s + ab)
    pool = O.build_pool(n_b)
    grids = np.zeros((len(pool) + 2, n_b, n_b), bool)
    for i, coords in enumerate(pool.values()):
        c = np.asarray(coords).reshape(-1, 2)
        grids[i, c[:, 0], c[:, 1]] = True
    for i in (len(pool), len(pool) + 1):  # random layouts, diagonal kept (sf/bench.py:54-62)
        grids[i] = rng.random((n_b, n_b)) < 0.2
        grids[i][np.arange(n_b), np.arange(n_b)] = True
    tab = PT.tables128_from_grids(grids, s, ab)
    gu = min(ab, 128)
    nsub = 128 // gu
    nt = -(-s // 128)
    for p in range(grids.shape[0]):
        want = grid_cells(grids[p], s, ab)
        csr, csc = decode(tab, p, s)
        np.testing.assert_array_equal(csr, want)
        np.testing.assert_array_equal(csc, want)
        # work = ceil(union / nsub) per tile (query side and key side)
        units_q = want.reshape(s // 16, s // gu, gu // 16).any(2)
        exp_f = sum(-(-int(units_q[t * 8 : (t + 1) * 8].any(0).sum()) // nsub) for t in range(nt))
        units_k = want.T.reshape(s // 16, s // gu, gu // 16).any(2)
        exp_b = sum(-(-int(units_k[t * 8 : (t + 1) * 8].any(0).sum()) // nsub) for t in range(nt))
        assert PT.tables128_work(tab, p) == (exp_f, exp_b)


def test_gather_turns_sparsity_into_fewer_tiles():
    """At attn_blk 64 / s 1024 a 90%-sparse random layout needs far fewer gathered tiles than 128-tiles touched."""
    s, ab = 1024, 64
    n_b = s // ab
    rng = np.random.default_rng(0)
    g = rng.random((n_b, n_b)) < 0.1
    g[np.arange(n_b), np.arange(n_b)] = True
    tab = PT.tables128_from_grids(g[None], s, ab)
    fwd, bwd = PT.tables128_work(tab, 0)
    dense = (s // 128) ** 2
    touched = int(g.reshape(8, 2, 8, 2).any(axis=(1, 3)).sum())
    assert fwd < touched <= dense and bwd < touched
