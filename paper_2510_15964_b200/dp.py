"""Data parallelism by batch.

The fine-tune step of sf/harness.py:396-417 averages per-sequence gradients
over the batch (`grads_mean = grads_sum / batch_size`, sf/harness.py:413-415)
and then runs one Adam update. With per-sequence mask scope every sequence is
independent, so the batch is split contiguously over ranks and the only
collective is ONE all-reduce (SUM, fp32) of the flat trainable-gradient buffer
per step -- 22 MB for OPT-1.3B LoRA. Adam then runs replicated and bit-identical
on every rank.

Each rank's engine produces the mean over its own shard; the hook rescales by
local/global before the SUM so ragged shards still give the global mean.
"""

from __future__ import annotations

from .errors import ConfigError


def shard_range(global_batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [start, stop) of rank `rank`; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"rank {rank} outside world of size {world}")
    if global_batch < world:
        raise ConfigError(f"global batch {global_batch} smaller than world size {world}: a rank would have no sequence")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def make_grad_hook(dist, global_batch: int, rank: int, world: int, group=None):
    """Hook for FinetuneEngine(grad_hook=...): turns this rank's shard-mean gradient into the
    global batch mean with one in-place all-reduce of the flat buffer. Returns None at world 1."""
    if world == 1:
        return None
    start, stop = shard_range(global_batch, rank, world)
    w = (stop - start) / global_batch

    def hook(flat_grad):
        flat_grad.mul_(w)
        dist.all_reduce(flat_grad, group=group)

    return hook


class BucketedGradSync:
    """The same global-mean reduction as make_grad_hook, issued per layer group DURING the backward (§8(e)):
    once a group's LoRA / BitFit column reductions have been written into the flat gradient buffer (the
    engine's _CgBatch flush), that slice is scaled and all-reduced on a dedicated communication stream, so the
    transfer overlaps the remaining layers' backward; `finish` reduces whatever the buckets did not cover and
    makes the compute stream wait for the collectives (Adam reads every gradient). NCCL collectives on that
    stream are captured into the engine's CUDA graph like its kernels. Deterministic: each element is reduced
    exactly once with the same operands as the single all-reduce."""

    def __init__(self, dist, global_batch: int, rank: int, world: int, group=None):
        start, stop = shard_range(global_batch, rank, world)
        self.w = (stop - start) / global_batch
        self.dist, self.group = dist, group
        self.stream = None
        self.done: list[tuple[int, int]] = []

    def begin(self) -> None:
        self.done = []

    def bucket(self, flat, lo: int, hi: int, producer_stream=None) -> None:
        if hi <= lo:
            return
        if flat.is_cuda:
            import torch

            if self.stream is None:
                self.stream = torch.cuda.Stream(device=flat.device)
            self.stream.wait_stream(torch.cuda.current_stream(flat.device))
            if producer_stream is not None:
                self.stream.wait_stream(producer_stream)
            with torch.cuda.stream(self.stream):
                v = flat[lo:hi]
                v.mul_(self.w)
                self.dist.all_reduce(v, group=self.group)
        else:
            v = flat[lo:hi]
            v.mul_(self.w)
            self.dist.all_reduce(v, group=self.group)
        self.done.append((lo, hi))

    def finish(self, flat) -> None:
        """Reduce the gaps between the issued buckets, then join the communication stream."""
        n, pos = flat.numel(), 0
        for lo, hi in sorted(self.done):
            if lo > pos:
                self.bucket(flat, pos, lo)
            pos = max(pos, hi)
        if pos < n:
            self.bucket(flat, pos, n)
        if flat.is_cuda and self.stream is not None:
            import torch

            torch.cuda.current_stream(flat.device).wait_stream(self.stream)
