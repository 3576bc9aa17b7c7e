"""Data-parallel step logic (paper_2510_15964_b200/dp.py) on CPU with gloo, world size 2.

Each rank computes the shard-mean gradients of its contiguous batch shard with the oracle
(the per-sequence fwd/bwd of sf/harness.py:401-411), packs them into a flat fp32 buffer, runs
the product hook (one all-reduce) and the product's flat Adam (autograd.adam_flat). The result
must equal the single-process full-batch step (oracle finetune_step): same mean gradients and,
on every rank, the same updated parameters."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sf_oracle as O

B_GLOBAL = 3  # ragged shards: 2 + 1


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    dims = O.Dims(32, 2, 64, 16, 2, 40, 8, 8)
    m = O.build_model(dims, seed=5, peft="lora")
    rng = np.random.default_rng(3)
    for ad in m.lora.values():
        ad["b"] += (rng.standard_normal(ad["b"].shape) * 0.02).astype(np.float32)
    toks = rng.integers(0, dims.vocab, size=(B_GLOBAL, dims.seq_len + 1))
    nm = np.ones(dims.n_blk, bool)
    nm[[1, 4, 5]] = False
    masks = [(["blockdiag", "dense"], nm), (["dense", "band1"], ~nm)]  # fixed sparse masks per layer
    return m, toks, masks


def _flat(grads: dict, names) -> torch.Tensor:
    return torch.from_numpy(np.concatenate([grads[n].ravel() for n in names]).astype(np.float32))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_15964_b200 import autograd as AG
    from paper_2510_15964_b200.dp import make_grad_hook, shard_range

    m, toks, prov = _problem()
    names = list(O.trainable_params(m))
    a, b = shard_range(B_GLOBAL, rank, world)
    gsum = None
    for seq in toks[a:b]:
        logits, cache = O.model_forward(m, seq[:-1], prov)
        g = O.model_backward(m, cache, O.loss_backward(logits, seq[1:]))
        f = _flat(g, names)
        gsum = f if gsum is None else gsum + f
    flat = gsum / (b - a)  # the engine's shard mean
    make_grad_hook(dist, B_GLOBAL, rank, world)(flat)
    p = torch.from_numpy(np.concatenate([O.trainable_params(m)[n].ravel() for n in names]).astype(np.float32))
    mom, vel = torch.zeros_like(flat, dtype=torch.float64), torch.zeros_like(flat, dtype=torch.float64)
    AG.adam_flat(p, flat.double(), mom, vel, 1e-3, 0.9, 0.999, 1e-8, 1)
    out[rank] = (flat.numpy().copy(), p.numpy().copy())
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_dp_allreduce_equals_full_batch_step():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    m, toks, prov = _problem()
    names = list(O.trainable_params(m))
    params = O.trainable_params(m)
    _, gmean, _ = O.finetune_step(m, toks, prov, params, {}, {}, 0, 1e-3)
    ref_g = _flat(gmean, names).numpy()
    ref_p = np.concatenate([params[n].ravel() for n in names])
    g0, p0 = out[0]
    g1, p1 = out[1]
    np.testing.assert_array_equal(g0, g1)  # all-reduce leaves identical buffers
    np.testing.assert_array_equal(p0, p1)  # replicated Adam stays bit-identical
    np.testing.assert_allclose(g0, ref_g, rtol=1e-5, atol=1e-6 * np.abs(ref_g).max())  # fp32 summation order
    np.testing.assert_allclose(p0, ref_p, rtol=1e-6, atol=1e-7)


def test_shard_range():
    from paper_2510_15964_b200.dp import shard_range
    from paper_2510_15964_b200.errors import ConfigError

    assert [shard_range(8, r, 4) for r in range(4)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    assert [shard_range(5, r, 2) for r in range(2)] == [(0, 3), (3, 5)]
    with pytest.raises(ConfigError):
        shard_range(1, 0, 2)
    with pytest.raises(ConfigError):
        shard_range(4, 2, 2)


def _bucket_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_15964_b200.dp import BucketedGradSync, make_grad_hook

    g = torch.Generator().manual_seed(rank)
    base = torch.randn(1000, generator=g)
    a = base.clone()
    make_grad_hook(dist, 5, rank, world)(a)
    b = base.clone()
    sync = BucketedGradSync(dist, 5, rank, world)
    sync.begin()
    sync.bucket(b, 700, 1000)  # layer groups in backward order (last layers first)
    sync.bucket(b, 300, 450)
    sync.finish(b)  # gaps [0, 300) and [450, 700)
    out[rank] = (a.numpy().copy(), b.numpy().copy(), sorted(sync.done))
    dist.destroy_process_group()


def test_bucketed_sync_equals_single_allreduce():
    """dp.BucketedGradSync (per layer group during the backward + the gaps at the end) reduces every element
    exactly once, with the same scaling: bit-identical to the single-all-reduce hook (gloo, world 2,
    ragged global batch 5 -> 3 + 2)."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_bucket_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        a, b, done = out[r]
        np.testing.assert_array_equal(a, b)
        assert done == [(0, 300), (300, 450), (450, 700), (700, 1000)]
    np.testing.assert_array_equal(out[0][1], out[1][1])


def _gpu_worker(rank, world, port, out, bucketed=False):
    """One rank of the device engine: its contiguous shard of the global batch, the production grad
    reduction (one all-reduce of the flat gradient buffer, or per-layer-group buckets during the backward;
    gloo here because both ranks share the GPU), replicated fused Adam."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2510_15964_b200.dp import BucketedGradSync, make_grad_hook, shard_range
    from paper_2510_15964_b200.engine import FinetuneEngine

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = dict(d=256, H=4, d_ff=1024, L=2, V=128, B=4, s=128, blk=16, attn_blk=32, r=8)
    model, state, prov = bench.build_workload(cfg, dev, 5, 0.5, 0.5)
    toks = torch.randint(0, cfg["V"], (cfg["B"], cfg["s"] + 1), generator=torch.Generator().manual_seed(9))
    a, b = shard_range(cfg["B"], rank, world) if world > 1 else (0, cfg["B"])
    hook = make_grad_hook(dist, cfg["B"], rank, world) if world > 1 and not bucketed else None
    sync = BucketedGradSync(dist, cfg["B"], rank, world) if world > 1 and bucketed else None
    eng = FinetuneEngine(model, state, prov, lr=1e-3, grad_hook=hook, grad_sync=sync)
    loss = eng.step(toks[a:b].to(dev))
    torch.cuda.synchronize()
    out[rank] = (eng.flat_grad.cpu().numpy().copy(), state.flat.cpu().numpy().copy(), float(loss))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_dp_engine_two_ranks_equals_single_rank():
    """The device fine-tune step data-parallel over two ranks (batch 4 -> 2 + 2, one all-reduce of the
    flat fp32 gradients, replicated Adam) equals the single-rank step over the whole batch: the same mean
    gradients up to fp32 summation order and bf16 kernel noise, bit-identical parameters on both ranks."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    mgr = mp.Manager()
    out2, out1, outb = mgr.dict(), mgr.dict(), mgr.dict()
    mp.spawn(_gpu_worker, args=(2, _free_port(), out2), nprocs=2, join=True)
    mp.spawn(_gpu_worker, args=(1, _free_port(), out1), nprocs=1, join=True)
    mp.spawn(_gpu_worker, args=(2, _free_port(), outb, True), nprocs=2, join=True)
    g0, p0, _ = out2[0]
    g1, p1, _ = out2[1]
    gs, ps, _ = out1[0]
    np.testing.assert_array_equal(g0, g1)
    np.testing.assert_array_equal(p0, p1)
    for r in range(2):  # bucketed reduction during the backward == one reduction after it, bit for bit
        np.testing.assert_array_equal(outb[r][0], out2[r][0])
        np.testing.assert_array_equal(outb[r][1], out2[r][1])
    scale = np.abs(gs).max()
    assert np.abs(g0 - gs).max() <= 1e-2 * scale  # per-item masks and kernels are identical; sums reordered
    assert np.abs(p0 - ps).max() <= 2 * 1e-3 + 1e-6  # Adam: at most one lr step apart per parameter


def test_bench_gpus_flag_fails_loudly_without_enough_gpus():
    """`bench.py --gpus N` launches N ranks itself; with fewer visible GPUs it exits non-zero at once (no silent
    single-GPU run), and a torchrun world that disagrees with --gpus is refused."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    import torch

    root = Path(__file__).resolve().parent.parent
    n = torch.cuda.device_count() + 1
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", str(n), "--steps", "1"], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 2 and "GPU" in r.stdout, (r.returncode, r.stdout, r.stderr[-500:])
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--steps", "1"], capture_output=True,
                       text=True, timeout=300, env=env)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stdout, (r.returncode, r.stdout)


def _nccl_capture_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    import bench
    from paper_2510_15964_b200.dp import BucketedGradSync
    from paper_2510_15964_b200.engine import FinetuneEngine

    cfg = dict(d=256, H=4, d_ff=1024, L=3, V=128, B=2, s=128, blk=16, attn_blk=32, r=8)
    toks = torch.randint(0, cfg["V"], (cfg["B"], cfg["s"] + 1), generator=torch.Generator().manual_seed(4)).to(dev)
    res = []
    for graph in (False, True):
        model, state, prov = bench.build_workload(cfg, dev, 6, 0.5, 0.5)
        eng = FinetuneEngine(model, state, prov, lr=1e-3, grad_sync=BucketedGradSync(dist, cfg["B"], rank, world))
        if graph:
            eng.capture(toks)
            eng.state.step = 0
            eng.replay()
        else:
            eng._step(toks)
            eng._finish()
        torch.cuda.synchronize()
        res.append((eng.flat_grad.cpu().numpy().copy(), eng.state.flat.cpu().numpy().copy()))
    out[rank] = res
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_bucketed_nccl_allreduce_is_captured_in_the_step_graph():
    """NCCL (world 1 on the one visible GPU): the per-layer-group all-reduces issued on the communication stream
    during the backward are captured into the engine's CUDA graph; a replay gives the eager step's gradients
    and parameters bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_nccl_capture_worker, args=(1, _free_port(), out), nprocs=1, join=True)
    (ge, pe), (gg, pg) = out[0]
    np.testing.assert_array_equal(ge, gg)
    np.testing.assert_array_equal(pe, pg)
