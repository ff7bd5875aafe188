"""Row-strip sharding: the multi-rank host logic on CPU with
gloo (world sizes 2 and 3), and the device halo path on one GPU with
virtual ranks (threads exchanging rows), both against the unsharded result.
"""
import os
import socket
import threading

import numpy as np
import pytest
import torch

from oracle import dwt_oracle as O
from paper_1704_08657_b200 import strips as S


def oracle_level_fn(wavelet, scheme, opt, up, down):
    """Level of the float64 oracle on [top; strip; bottom] cropped to the
    strip's component rows (the periodic wrap of the tall image never reaches
    them: every output row depends on rows up..down around it)."""
    def fn(cur, top, bottom):
        tall = torch.cat([top, cur, bottom]).double().numpy()
        res = O.transform(wavelet, scheme, O.split(tall), opt)
        h2 = cur.shape[0] // 2
        return [torch.from_numpy(np.ascontiguousarray(r[up:up + h2])) for r in res]
    return fn


def oracle_pair_fn(wavelet, scheme, opt, up, down):
    """Levels 1 and 2 of the float64 oracle on [top; strip; bottom] with the
    fused pair's 6*up / 6*down halo rows, cropped to the strip's rows."""
    def fn(cur, top, bottom):
        tall = torch.cat([top, cur, bottom]).double().numpy()
        r1 = O.transform(wavelet, scheme, O.split(tall), opt)
        h2 = cur.shape[0] // 2
        det1 = [torch.from_numpy(np.ascontiguousarray(r[3 * up:3 * up + h2])) for r in r1[1:]]
        ll1 = r1[0]
        s0 = (3 * up) % 2  # first LL_1 row of an even global row
        n = ll1.shape[0] - s0
        ll1 = ll1[s0:s0 + n - n % 2]
        r2 = O.transform(wavelet, scheme, O.split(ll1), opt)
        o2 = (3 * up - s0) // 2
        lvl2 = [torch.from_numpy(np.ascontiguousarray(r[o2:o2 + h2 // 2])) for r in r2]
        return det1, lvl2
    return fn


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, args, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wavelet, scheme, opt, W, Hs, levels, pair = args
        img = O.random_image(W, Hs * world, 1, np.float64)
        strip = torch.from_numpy(img[rank * Hs:(rank + 1) * Hs].copy())
        r = 2 if wavelet == "cdf97" else 1
        out = S.forward_mallat_strips(oracle_level_fn(wavelet, scheme, opt, r, r), strip, levels, r, r,
                                      S.HaloExchange(),
                                      pair_fn=oracle_pair_fn(wavelet, scheme, opt, r, r) if pair else None)
        gathered = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(gathered, out)
        if rank == 0:
            g = S.assemble_mallat(gathered, levels)
            truth = O.pyramid(wavelet, scheme, img, levels, opt)
            q.put(float(np.max(np.abs(g.numpy() - truth))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("wavelet,scheme,opt", [("cdf97", "nonseparable-lifting", True),
                                                ("cdf53", "separable-lifting", False)])
@pytest.mark.parametrize("pair", [False, True])
def test_gloo_strip_pyramid_equals_full_image(world, wavelet, scheme, opt, pair):
    """Strip pyramid over gloo ranks = the full-image oracle pyramid; with
    `pair`, levels 1+2 come from one 6*up / 6*down-row halo exchange (the
    fused level pair's data flow)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    args = (wavelet, scheme, opt, 32, 32, 3, pair)
    procs = [ctx.Process(target=_worker, args=(r, world, port, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) < 1e-12


def _pitched_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        strip = torch.arange(60.0).reshape(10, 6) + 1000 * rank
        # the C++ driver's halo rows from level 3 on: w floats of a wider pitch
        buf = torch.full((8, 16), -1.0)
        top, bottom = buf[:4, :6], buf[4:7, :6]
        assert not top.is_contiguous()
        S.HaloExchange()(strip, 4, 3, top=top, bottom=bottom)
        prev, nxt = S.ring_neighbours(rank, world)
        ok = (torch.equal(top, torch.arange(60.0).reshape(10, 6)[-4:] + 1000 * prev) and
              torch.equal(bottom, torch.arange(60.0).reshape(10, 6)[:3] + 1000 * nxt) and
              bool((buf[:, 6:] == -1).all()))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchange_into_pitched_views(world):
    """HaloExchange with world > 1 fills non-contiguous (pitched) halo views
    row by row and leaves the rest of the pitch alone."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pitched_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(ok for _, ok in res), res


def test_exchange_into_given_buffers():
    """HaloExchange receives into caller buffers (the C++ strip driver's
    callback contract); single rank: periodic wrap."""
    strip = torch.arange(40.0).reshape(10, 4)
    top, bottom = torch.empty(3, 4), torch.empty(2, 4)
    t, b = S.HaloExchange()(strip, 3, 2, top=top, bottom=bottom)
    assert t is top and b is bottom
    assert torch.equal(top, strip[-3:]) and torch.equal(bottom, strip[:2])


def test_single_rank_exchange_is_periodic_wrap():
    img = O.random_image(32, 32, 5, np.float64)
    out = S.forward_mallat_strips(oracle_level_fn("cdf97", "nonseparable-lifting", True, 2, 2),
                                  torch.from_numpy(img.copy()), 3, 2, 2, S.HaloExchange())
    truth = O.pyramid("cdf97", "nonseparable-lifting", img, 3, True)
    assert np.max(np.abs(out.numpy() - truth)) < 1e-12


def test_strip_validation_and_assembly():
    with pytest.raises(ValueError):
        S.check_strip(2, 8, 2, 2)  # thinner than its 4-row halo
    with pytest.raises(ValueError):
        S.check_strip(6, 7, 1, 1)
    assert S.ring_neighbours(0, 4) == (3, 1)
    assert S.ring_neighbours(3, 4) == (2, 0)


class VirtualRing:
    """N ranks as threads in one process: each publishes its strip at every
    level and reads its neighbours' rows (device tensors, same GPU)."""

    def __init__(self, world):
        self.world = world
        self.slots = [None] * world
        self.barrier = threading.Barrier(world)

    def exchange_for(self, rank):
        def ex(strip, top_rows, bottom_rows):
            self.slots[rank] = strip
            self.barrier.wait()
            prev, nxt = S.ring_neighbours(rank, self.world)
            top = self.slots[prev][-top_rows:].contiguous()
            bottom = self.slots[nxt][:bottom_rows].contiguous()
            torch.cuda.synchronize()
            self.barrier.wait()
            return top, bottom
        return ex


@pytest.mark.gpu
@pytest.mark.parametrize("tma,pair", [("0", False), ("2", False), ("1", True)])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("wavelet,scheme,opt", [("cdf97", "nonseparable-lifting", True),
                                                ("cdf97", "separable-convolution", False),
                                                ("dd137", "nonseparable-lifting", True)])
def test_gpu_strip_kernels_equal_single_gpu_pyramid(cuda, world, wavelet, scheme, opt, tma, pair):
    """The halo-row path of the fused kernel reproduces the single-GPU
    pyramid bit for bit (same arithmetic; halo rows are the same data), with
    register prefetch (DWT2D_TMA=0), TMA-staged rows (=2), and with levels
    1+2 as one fused pass from 6*up/6*down halo rows (pair)."""
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan(wavelet, scheme, optimized=opt).tune(tma=int(tma))
    up, down = plan.info["reach_up"], plan.info["reach_down"]
    W, Hs, L = 256, 128, 4
    img = torch.from_numpy(O.random_image(W, Hs * world, 3)).to(cuda)
    full = plan.forward_mallat(img, L)
    ring = VirtualRing(world)
    outs = [None] * world
    errors = []

    def run(rank):
        try:
            torch.cuda.set_device(cuda)
            strip = img[rank * Hs:(rank + 1) * Hs].contiguous()
            outs[rank] = S.forward_mallat_strips(S.gpu_level_fn(plan), strip, L, up, down,
                                                 ring.exchange_for(rank),
                                                 pair_fn=S.gpu_pair_fn(plan) if pair else None)
            torch.cuda.synchronize()
        except Exception as e:  # surfaced below
            errors.append(e)
            ring.barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    g = S.assemble_mallat(outs, L)
    assert torch.equal(g, full.cpu())


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("wavelet,scheme,opt", [("cdf97", "nonseparable-lifting", True),
                                                ("cdf53", "separable-lifting", False),
                                                ("dd137", "nonseparable-lifting", True)])
@pytest.mark.parametrize("pair,own_stream", [("1", False), ("0", False), ("1", True)])
def test_gpu_strip_driver_equals_single_gpu_pyramid(cuda, world, wavelet, scheme, opt, pair, own_stream):
    """The C++ strip-pyramid driver (dwt2d_forward_mallat_strip) with a
    Python halo-exchange callback reproduces the single-GPU pyramid bit for
    bit: world 1 without a callback (periodic wrap inside the strip), 2 and
    4 virtual ranks as threads; with and without the fused level pair."""
    import paper_1704_08657_b200 as dwt
    plan = dwt.Plan(wavelet, scheme, optimized=opt).tune(pair=int(pair))
    W, Hs, L = 256, 128, 4
    img = torch.from_numpy(O.random_image(W, Hs * world, 3)).to(cuda)
    full = plan.forward_mallat(img, L)
    if world == 1:
        got = S.gpu_forward_mallat(plan, img, L)
        torch.cuda.synchronize()
        assert torch.equal(got, full)
        return
    ring = VirtualRing(world)
    outs = [None] * world
    errors = []

    def run(rank):
        try:
            torch.cuda.set_device(cuda)
            ex = ring.exchange_for(rank)

            def fill(cur, tr, br, top, bottom):
                t, b = ex(cur, tr, br)
                top.copy_(t)
                bottom.copy_(b)
            strip = img[rank * Hs:(rank + 1) * Hs].contiguous()
            # own_stream: the library runs on a stream that is not torch's
            # current one; the callback's copies must still be ordered with it
            st = torch.cuda.Stream() if own_stream else None
            if st is not None:
                st.wait_stream(torch.cuda.current_stream())
            outs[rank] = S.gpu_forward_mallat(plan, strip, L, exchange=fill, stream=st)
            torch.cuda.synchronize()
        except Exception as e:  # surfaced below
            errors.append(e)
            ring.barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    assert torch.equal(S.assemble_mallat(outs, L), full.cpu())


def _gpu_worker(rank, world, port, q):
    import torch.distributed as dist
    import paper_1704_08657_b200 as dwt
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
        W, Hs, L = 512, 256, 4
        img = torch.from_numpy(O.random_image(W, Hs * world, 7)).cuda()
        ex = S.HaloExchange()

        def exchange(cur, tr, br, top, bottom):  # gloo moves host tensors
            t, b = ex(cur.cpu(), tr, br)
            top.copy_(t)
            bottom.copy_(b)

        out = S.gpu_forward_mallat(plan, img[rank * Hs:(rank + 1) * Hs].contiguous(), L, exchange=exchange)
        torch.cuda.synchronize()
        gathered = [torch.empty((Hs, W)) for _ in range(world)]
        dist.all_gather(gathered, out.cpu())
        if rank == 0:
            full = plan.forward_mallat(img, L).cpu()
            q.put(bool(torch.equal(S.assemble_mallat(gathered, L), full)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_gpu_strip_driver_across_processes(world):
    """The C++ strip driver in separate processes (one rank each, sharing one
    GPU) with a real torch.distributed exchange (gloo over host copies):
    bit-identical to the single-GPU pyramid."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True
