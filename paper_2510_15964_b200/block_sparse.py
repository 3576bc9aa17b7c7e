"""Block-sparse attention on the B200 (drop-in for sf/block_sparse.py).

Hot path: `attention_forward` / `attention_backward` run the fused
SDD -> sparse softmax -> DSD chain (and its backward) in the tcgen05 kernels of
csrc/attn_sm100.cu, walking each (item, head)'s pool pattern through the gathered
128-tile tables (patterns.tables128_from_grids): only the active blocks' keys
(forward, dQ) or queries (dK/dV) are loaded and multiplied. The probabilities
are never materialised (the cache holds O and the row LSE).

There is one implementation. The kernels take the fused projection output
([M, 3d], q | k | v column blocks) at head_dim 64 or 128; other operands (separate
q/k/v, other head dims) are staged into that layout with the head dimension
zero-padded to 64 / 128 -- zero columns change neither QK^T nor the used part of
P.V -- and the explicit `scale` keeps 1/sqrt(hd) of the true head dim.

The reference's materialising operators (`sdd`, `sparse_softmax`, `dsd` and
their backward, over `BlockSparseMatrix`) are kept with the same signatures
for API parity and debugging; they run as batched device tensor ops over the
gathered active blocks and are not used by the training step.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from .errors import LayoutError, UnsupportedError
from .patterns import DevicePool

Coord = tuple[int, int]


# ---------------------------------------------------------------- fused hot path


def _padded_hd(hd: int) -> int:
    if hd <= 64:
        return 64
    if hd <= 128:
        return 128
    raise UnsupportedError(f"head_dim {hd} > 128 unsupported by the tcgen05 attention kernels")


def _is_fused(q, k, v, ld: int, d: int) -> bool:
    return ld == 3 * d and k.data_ptr() == q.data_ptr() + 2 * d and v.data_ptr() == q.data_ptr() + 4 * d


def _stage(ts, M: int, H: int, hd: int, hdp: int) -> torch.Tensor:
    """[M, len(ts) * H * hdp] bf16 with tensor t's head h at block t, columns h*hdp .. h*hdp + hd (rest 0)."""
    out = torch.zeros(M, len(ts), H, hdp, dtype=torch.bfloat16, device=ts[0].device)
    for i, t in enumerate(ts):
        out[:, i, :, :hd] = t[:M, : H * hd].reshape(M, H, hd)
    return out.view(M, len(ts) * H * hdp)


def _check_tables(dpool: DevicePool, s: int):
    if dpool.tables is None or dpool.seq_len != s:
        raise LayoutError(f"device pool tables were built for seq_len {dpool.seq_len}, not {s}")


def attention_forward(q, k, v, ld: int, n_items: int, s: int, H: int, hd: int, pidx: torch.Tensor, item_stride: int,
                      dpool: DevicePool, scale: float, out: torch.Tensor | None = None):
    """Non-causal block-sparse attention for all (item, head): returns (O bf16 [n_items*s, H*hd], lse fp32 [n_items, H, s])."""
    _check_tables(dpool, s)
    dev = q.device
    M, d = n_items * s, H * hd
    o = out if out is not None else torch.empty(M, d, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(n_items, H, s, dtype=torch.float32, device=dev)
    if _is_fused(q, k, v, ld, d) and hd in (64, 128):
        _abi.call("lx_bsattn_fwd_tc", q.data_ptr(), ld, n_items, s, H, hd, pidx.data_ptr(), item_stride,
                  dpool.tables.data_ptr(), dpool.gather_rows, float(scale), o.data_ptr(), o.stride(0), lse.data_ptr(),
                  _abi.stream_handle(dev))
        return o, lse
    hdp = _padded_hd(hd)
    qkv = _stage([q, k, v], M, H, hd, hdp)
    op = torch.empty(M, H * hdp, dtype=torch.bfloat16, device=dev)
    _abi.call("lx_bsattn_fwd_tc", qkv.data_ptr(), qkv.stride(0), n_items, s, H, hdp, pidx.data_ptr(), item_stride,
              dpool.tables.data_ptr(), dpool.gather_rows, float(scale), op.data_ptr(), op.stride(0), lse.data_ptr(),
              _abi.stream_handle(dev))
    o.view(M, H, hd).copy_(op.view(M, H, hdp)[:, :, :hd])
    return o, lse


def attention_backward(q, k, v, o, d_o, ld: int, n_items: int, s: int, H: int, hd: int, pidx, item_stride: int,
                       dpool: DevicePool, scale: float, lse, dq, dk, dv):
    """dq/dk/dv (bf16) of the fused forward; deterministic (fixed accumulation order)."""
    _check_tables(dpool, s)
    dev = q.device
    M, d = n_items * s, H * hd
    delta = torch.empty(n_items, H, s, dtype=torch.float32, device=dev)
    if d_o.stride(0) != o.stride(0):
        raise LayoutError("attention_backward expects o and d_o with the same row stride")
    fused = (_is_fused(q, k, v, ld, d) and hd in (64, 128) and dk.data_ptr() == dq.data_ptr() + 2 * d
             and dv.data_ptr() == dq.data_ptr() + 4 * d and dk.stride(0) == dq.stride(0) == dv.stride(0) >= 3 * d)
    if fused:
        # dqkv may be the K-extended [M, 3d + kx] operand of the projection input-grad GEMM (row stride dq.stride(0))
        ws = torch.empty(n_items * H * (hd + 8 * ((s + 127) // 128)), dtype=torch.float32, device=dev)
        _abi.call("lx_bsattn_bwd_tc", q.data_ptr(), ld, dq.stride(0), o.data_ptr(), d_o.data_ptr(), o.stride(0), n_items, s, H,
                  hd, pidx.data_ptr(), item_stride, dpool.tables.data_ptr(), dpool.gather_rows, float(scale), lse.data_ptr(),
                  delta.data_ptr(), ws.data_ptr(), dq.data_ptr(), _abi.stream_handle(dev))
        return
    hdp = _padded_hd(hd)
    qkv = _stage([q, k, v], M, H, hd, hdp)
    od = _stage([o, d_o], M, H, hd, hdp)
    dqkv = torch.empty(M, 3 * H * hdp, dtype=torch.bfloat16, device=dev)
    ws = torch.empty(n_items * H * (hdp + 8 * ((s + 127) // 128)), dtype=torch.float32, device=dev)
    _abi.call("lx_bsattn_bwd_tc", qkv.data_ptr(), qkv.stride(0), dqkv.stride(0), od.data_ptr(), od[:, H * hdp :].data_ptr(),
              od.stride(0), n_items, s, H, hdp, pidx.data_ptr(), item_stride, dpool.tables.data_ptr(), dpool.gather_rows,
              float(scale), lse.data_ptr(), delta.data_ptr(), ws.data_ptr(), dqkv.data_ptr(), _abi.stream_handle(dev))
    g = dqkv.view(M, 3, H, hdp)
    for i, dst in enumerate((dq, dk, dv)):
        dst[:M, :d].view(M, H, hd).copy_(g[:, i, :, :hd])


# ---------------------------------------------------------------- reference-API operators


@dataclass
class BlockSparseMatrix:
    """Block-sparse s x s matrix over an n_b x n_b grid (sf/block_sparse.py:22-36)."""

    n_b: int
    blk: int
    coords: tuple[Coord, ...]
    blocks: torch.Tensor  # (len(coords), blk, blk), layout order

    def to_dense(self) -> torch.Tensor:
        s = self.n_b * self.blk
        out = torch.zeros(s, s, dtype=self.blocks.dtype, device=self.blocks.device)
        c = torch.as_tensor(self.coords, device=self.blocks.device).reshape(-1, 2)
        view = out.view(self.n_b, self.blk, self.n_b, self.blk).permute(0, 2, 1, 3)
        view[c[:, 0], c[:, 1]] = self.blocks
        return out


def _coords_t(coords, n_b, device):
    c = torch.as_tensor(np.asarray(coords, dtype=np.int64).reshape(-1, 2), device=device)
    if c.numel() and (int(c.min()) < 0 or int(c.max()) >= n_b):
        raise LayoutError(f"block outside {n_b}x{n_b} grid")
    return c


def sdd(q, k, coords, blk: int, scale: float, counter=None) -> BlockSparseMatrix:
    """sf/block_sparse.py:47-60."""
    s, hd = q.shape
    n_b = s // blk
    if s != n_b * blk:
        raise LayoutError(f"sequence length {s} != n_b*blk = {n_b}*{blk}")
    c = _coords_t(coords, n_b, q.device)
    qb = q.reshape(n_b, blk, hd)[c[:, 0]]
    kb = k.reshape(n_b, blk, hd)[c[:, 1]]
    if counter is not None:
        counter.add(len(c) * blk * blk * hd)
    return BlockSparseMatrix(n_b, blk, tuple(map(tuple, np.asarray(coords).reshape(-1, 2).tolist())), (qb @ kb.transpose(1, 2)) * scale)


def sparse_softmax(m: BlockSparseMatrix) -> BlockSparseMatrix:
    """sf/block_sparse.py:81-99."""
    c = _coords_t(m.coords, m.n_b, m.blocks.device)
    br = c[:, 0]
    covered = torch.zeros(m.n_b, dtype=torch.bool, device=m.blocks.device)
    covered[br] = True
    if not bool(covered.all()):
        raise LayoutError("block-row has no active blocks (pattern pool violation)")
    rmax = torch.full((m.n_b, m.blk), -torch.inf, dtype=m.blocks.dtype, device=m.blocks.device)
    rmax = rmax.index_reduce(0, br, m.blocks.amax(2), "amax")
    e = torch.exp(m.blocks - rmax[br][:, :, None])
    den = torch.zeros(m.n_b, m.blk, dtype=m.blocks.dtype, device=m.blocks.device).index_add(0, br, e.sum(2))
    return BlockSparseMatrix(m.n_b, m.blk, m.coords, e / den[br][:, :, None])


def sparse_softmax_backward(p: BlockSparseMatrix, d_blocks):
    """sf/block_sparse.py:102-113."""
    br = _coords_t(p.coords, p.n_b, p.blocks.device)[:, 0]
    inner = torch.zeros(p.n_b, p.blk, dtype=p.blocks.dtype, device=p.blocks.device).index_add(0, br, (d_blocks * p.blocks).sum(2))
    return p.blocks * (d_blocks - inner[br][:, :, None])


def dsd(p: BlockSparseMatrix, v, counter=None):
    """sf/block_sparse.py:116-126."""
    s, hd = v.shape
    if s != p.n_b * p.blk:
        raise LayoutError(f"value rows {s} != grid {p.n_b}*{p.blk}")
    c = _coords_t(p.coords, p.n_b, v.device)
    prod = p.blocks @ v.reshape(p.n_b, p.blk, hd)[c[:, 1]]
    out = torch.zeros(p.n_b, p.blk, hd, dtype=prod.dtype, device=v.device).index_add(0, c[:, 0], prod)
    if counter is not None:
        counter.add(len(c) * p.blk * p.blk * hd)
    return out.reshape(s, hd)


def dsd_backward(p: BlockSparseMatrix, v, d_out):
    """sf/block_sparse.py:129-137."""
    s, hd = v.shape
    c = _coords_t(p.coords, p.n_b, v.device)
    g = d_out.reshape(p.n_b, p.blk, hd)[c[:, 0]]
    d_blocks = g @ v.reshape(p.n_b, p.blk, hd)[c[:, 1]].transpose(1, 2)
    dv = torch.zeros(p.n_b, p.blk, hd, dtype=v.dtype, device=v.device).index_add(0, c[:, 1], p.blocks.transpose(1, 2) @ g)
    return d_blocks, dv.reshape(s, hd)


def sdd_backward(d_blocks, q, k, coords, blk: int, scale: float):
    """sf/block_sparse.py:63-71."""
    s, hd = q.shape
    n_b = s // blk
    c = _coords_t(coords, n_b, q.device)
    g = d_blocks * scale
    dq = torch.zeros(n_b, blk, hd, dtype=q.dtype, device=q.device).index_add(0, c[:, 0], g @ k.reshape(n_b, blk, hd)[c[:, 1]])
    dk = torch.zeros(n_b, blk, hd, dtype=k.dtype, device=k.device).index_add(0, c[:, 1], g.transpose(1, 2) @ q.reshape(n_b, blk, hd)[c[:, 0]])
    return dq.reshape(s, hd), dk.reshape(s, hd)


def dense_masked_attention(q, k, v, coords, blk: int, scale: float):
    """sf/block_sparse.py:140-150 (float64 -inf-masked oracle on device)."""
    s = q.shape[0]
    mask = torch.full((s, s), -torch.inf, dtype=torch.float64, device=q.device)
    for br, bc in np.asarray(coords).reshape(-1, 2):
        mask[br * blk : (br + 1) * blk, bc * blk : (bc + 1) * blk] = 0.0
    sc = (q.double() @ k.double().T) * scale + mask
    return torch.softmax(sc, dim=1) @ v.double()
