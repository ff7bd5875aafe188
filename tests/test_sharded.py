"""The library's device-side sharded pyramid (dwt2d_shard_*,
dwt2d_forward_mallat_sharded): row strips in a ring,
halo rows pushed into the neighbours' exchange windows over peer memory.

Only one GPU is available to this build, so rings are exercised with
virtual ranks: several shards on device 0 (same process: peer pointers are
plain device pointers; separate processes: CUDA IPC handles of the windows,
exchanged over gloo). Every result is compared bit for bit with the
single-GPU pyramid of the whole image (the halo rows are the same data and
the arithmetic per output row does not depend on the strip split).
"""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import dwt_oracle as O
from paper_1704_08657_b200 import strips as S

pytestmark = pytest.mark.gpu


def _full_and_strips(W, Hs, world, seed=3):
    from paper_1704_08657_b200.synth import random_image
    img = random_image(W, Hs * world, seed, device="cuda")
    return img, [img[r * Hs:(r + 1) * Hs].contiguous() for r in range(world)]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("wavelet,scheme,opt,pair", [("cdf97", "nonseparable-lifting", True, 1),
                                                     ("cdf97", "nonseparable-lifting", True, 0),
                                                     ("cdf53", "separable-lifting", False, 1),
                                                     ("cdf97", "separable-convolution", False, 1),
                                                     ("dd137", "nonseparable-lifting", True, 1)])
def test_sharded_driver_equals_single_gpu_pyramid(cuda, world, wavelet, scheme, opt, pair):
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan(wavelet, scheme, optimized=opt).tune(pair=pair)
    W, Hs, L = 512, 256, 5
    img, strips = _full_and_strips(W, Hs, world)
    full = plan.forward_mallat(img, L)
    for _ in range(3):  # repeated pyramids: the done/arrival counters carry over
        outs = S.forward_mallat_sharded(plan, strips, L)
        torch.cuda.synchronize()
        assert torch.equal(S.assemble_mallat(outs, L), full.cpu())


def test_sharded_interior_split_and_deep_levels(cuda):
    """Tall strips (interior/border split on every level), strips that get
    as thin as their halo at the last level, pitched outputs."""
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    W, Hs, world, L = 1024, 1024, 4, 8  # level 8: 8-row strips, 4-row halo
    img, strips = _full_and_strips(W, Hs, world, 5)
    full = plan.forward_mallat(img, L)
    big = [torch.zeros((Hs, W + 64), device=cuda) for _ in range(world)]
    outs = S.forward_mallat_sharded(plan, strips, L, outs=[b[:, 32:32 + W] for b in big])
    torch.cuda.synchronize()
    assert torch.equal(S.assemble_mallat([o.contiguous() for o in outs], L), full.cpu())
    assert all(bool((b[:, :32] == 0).all()) for b in big)


def test_sharded_per_rank_calls_on_separate_streams(cuda):
    """Each rank enqueues its whole pyramid (dwt2d_shard_forward_mallat) on
    its own stream, rank after rank from one thread: the device-side waits
    resolve across streams."""
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    W, Hs, world, L = 512, 256, 3, 5
    img, strips = _full_and_strips(W, Hs, world, 7)
    full = plan.forward_mallat(img, L)
    torch.cuda.synchronize()
    shards = [S.Shard(plan, W, Hs, L, r, world) for r in range(world)]
    S.connect_ring(shards)
    streams = [torch.cuda.Stream() for _ in range(world)]
    for it in range(2):
        outs = [sh.forward_mallat(st_, stream=stream) for sh, st_, stream in zip(shards, strips, streams)]
        torch.cuda.synchronize()
        assert torch.equal(S.assemble_mallat(outs, L), full.cpu()), it
    assert all(sh.status() == 0 for sh in shards)


def _fresh_process_per_rank(q):
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    W, Hs, world, L = 2048, 1024, 2, 8
    img, strips = _full_and_strips(W, Hs, world, 13)
    shards = [S.Shard(plan, W, Hs, L, r, world) for r in range(world)]
    S.connect_ring(shards)
    streams = [torch.cuda.Stream() for _ in range(world)]
    outs = [sh.forward_mallat(s, stream=st) for sh, s, st in zip(shards, strips, streams)]
    torch.cuda.synchronize()
    full = plan.forward_mallat(img, L)
    q.put(bool(torch.equal(S.assemble_mallat(outs, L), full.cpu())))


def test_sharded_per_rank_calls_in_fresh_process():
    """Rank after rank from one thread in a process that has launched none
    of the level kernels yet: every kernel must already be loaded when the
    first rank's halo wait spins (lazy loading at a later launch would wait
    for it: a deadlock)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_fresh_process_per_rank, args=(q,))
    p.start()
    p.join(120)
    assert p.exitcode == 0
    assert q.get(timeout=10) is True


def test_sharded_graph_capture_and_replay(cuda):
    """The strip pyramids (pushes, waits and levels) captured in one CUDA
    graph replay correctly (the counters live on the device)."""
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    W, Hs, world, L = 512, 512, 4, 6
    img, strips = _full_and_strips(W, Hs, world, 9)
    full = plan.forward_mallat(img, L).cpu()
    outs = [torch.empty_like(s) for s in strips]
    S.forward_mallat_sharded(plan, strips, L, outs=outs)  # warm-up: shards created, tables uploaded
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        S.forward_mallat_sharded(plan, strips, L, outs=outs, streams=[s] * world)
    for _ in range(3):
        for o in outs:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(S.assemble_mallat(outs, L), full)


def test_sharded_world1_and_validation(cuda):
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    img, _ = _full_and_strips(256, 256, 1)
    sh = S.Shard(plan, 256, 256, 4)  # ring of one: no connect needed
    assert torch.equal(sh.forward_mallat(img), plan.forward_mallat(img, 4))
    with pytest.raises(dwt.DwtError):  # level 6 of a 64-row strip: 2 rows, thinner than its 4-row halo
        S.Shard(plan, 256, 64, 6, 0, 4)
    lone = S.Shard(plan, 256, 256, 4, 0, 2)
    with pytest.raises(ValueError):  # not connected
        lone.forward_mallat(img)
    with pytest.raises(ValueError):
        S.Shard(plan, 256, 256, 4, 2, 2)  # rank outside the ring
    inv = dwt.Plan("cdf97", "inverse-lifting")
    with pytest.raises(ValueError):
        S.Shard(inv, 256, 256, 4)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_config4_65536_sharded_equals_single_gpu(cuda, world):
    """configs[4]: the 65536^2 image as `world` row strips (virtual ranks on
    one GPU), 8 levels: bit-identical to the single-GPU pyramid."""
    import paper_1704_08657_b200 as dwt
    from paper_1704_08657_b200.synth import random_image
    n, L = 65536, 8
    plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
    img = random_image(n, n, 1, device="cuda")
    full = plan.forward_mallat(img, L)
    Hs = n // world
    strips = [img[r * Hs:(r + 1) * Hs] for r in range(world)]  # row views: contiguous
    outs = S.forward_mallat_sharded(plan, strips, L)
    torch.cuda.synchronize()
    # compare each strip's bands with the full pyramid's rows of that strip
    w, h = n, n
    for lvl in range(L):
        w2, h2 = w // 2, h // 2
        hl = (Hs >> lvl) // 2
        for r, o in enumerate(outs):
            hs = Hs >> lvl
            assert torch.equal(o[:hl, w2:w], full[r * hl:(r + 1) * hl, w2:w]), (lvl, r)
            assert torch.equal(o[hl:hs, :w], full[h2 + r * hl:h2 + (r + 1) * hl, :w]), (lvl, r)
            if lvl == L - 1:
                assert torch.equal(o[:hl, :w2], full[r * hl:(r + 1) * hl, :w2]), r
        w, h = w2, h2
    del outs, full, img
    torch.cuda.empty_cache()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist
    import paper_1704_08657_b200 as dwt
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
        W, Hs, L = 512, 256, 5
        img, strips = _full_and_strips(W, Hs, world, 11)
        sh = S.dist_shard(plan, W, Hs, L)
        for _ in range(2):
            out = sh.forward_mallat(strips[rank])
            torch.cuda.synchronize()
        gathered = [torch.empty((Hs, W)) for _ in range(world)]
        dist.all_gather(gathered, out.cpu())
        dist.barrier()
        if rank == 0:
            full = plan.forward_mallat(img, L).cpu()
            q.put(bool(torch.equal(S.assemble_mallat(gathered, L), full)))
        del sh
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_across_processes_ipc(world):
    """One rank per process (sharing one GPU), exchange windows mapped with
    CUDA IPC handles: bit-identical to the single-GPU pyramid."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True
