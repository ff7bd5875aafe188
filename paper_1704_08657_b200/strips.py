"""Row-strip sharding of the Mallat pyramid across GPUs.

A W x (N*H) image is split into N row strips, one per rank. Level l of the
pyramid on rank r needs, besides its own strip of LL_{l-1}, the 2*up image
rows directly above the strip (the previous rank's last rows) and the
2*down rows directly below (the next rank's first rows); periodic extension
closes the ring (rank N-1 <-> rank 0). `up`/`down` are the plan's component
-row reach (2 and 2 for CDF 9/7: 4 image rows, 256 KiB per side at W=16384).

Per level:  exchange halo rows with both ring neighbours (one batched
send/recv round: NCCL over NVLink between GPUs, gloo on CPU)  ->  run the
level on the strip with the halos as row sources (dwt2d_forward_level_strip,
the same fused kernel as the single-GPU path)  ->  the strip of LL_l is the
next level's input. Output per rank is a "strip Mallat" buffer (the rank's
rows of every band, in the Mallat quadrant layout of its strip);
`assemble_mallat` puts N of them back into the global layout.

The exchange is the only collective; the level math never crosses ranks.
"""
from __future__ import annotations

from typing import Callable, Sequence


def ring_neighbours(rank: int, world: int) -> tuple[int, int]:
    return (rank - 1) % world, (rank + 1) % world


def check_strip(h: int, w: int, up: int, down: int) -> None:
    if h % 2 or w % 2 or h <= 0 or w <= 0:
        raise ValueError("strip sides must be positive and even")
    if h < 2 * up or h < 2 * down:
        raise ValueError(f"strip of {h} rows is thinner than its halo ({2 * up}/{2 * down} rows); "
                         "use fewer ranks or levels")


class HaloExchange:
    """Ring halo exchange over torch.distributed (any backend)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def __call__(self, strip, top_rows: int, bottom_rows: int, top=None, bottom=None):
        """Returns (top, bottom): the rows above and below `strip` in the
        global (periodic) image, received into `top`/`bottom` if given."""
        if self.world == 1:  # periodic wrap of the only strip
            if top is None:
                return strip[-top_rows:], strip[:bottom_rows]
            top.copy_(strip[-top_rows:])
            bottom.copy_(strip[:bottom_rows])
            return top, bottom
        import torch
        dist = self.dist
        prev, nxt = ring_neighbours(self.rank, self.world)
        # receive into contiguous buffers: backends move numel() packed
        # elements from data_ptr(), so a pitched view (the library's halo
        # rows are w floats of a wider pitch from level 3 on) would get
        # rows 1.. misplaced; such views are filled by a copy afterwards
        rtop = top if top is not None and top.is_contiguous() else torch.empty(
            (top_rows, strip.shape[1]), dtype=strip.dtype, device=strip.device)
        rbot = bottom if bottom is not None and bottom.is_contiguous() else torch.empty(
            (bottom_rows, strip.shape[1]), dtype=strip.dtype, device=strip.device)
        # Post order matters when prev == next (2 ranks): messages between one
        # pair of ranks match in posting order, so sends go [to prev: my first
        # rows, to next: my last rows] and receives [from next: bottom, from
        # prev: top] — the k-th send of one rank meets the k-th receive of the
        # other for any world size.
        ops = [
            dist.P2POp(dist.isend, strip[:bottom_rows].contiguous(), prev, self.group),
            dist.P2POp(dist.isend, strip[-top_rows:].contiguous(), nxt, self.group),
            dist.P2POp(dist.irecv, rbot, nxt, self.group),
            dist.P2POp(dist.irecv, rtop, prev, self.group),
        ]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if top is None:
            top = rtop
        elif top.data_ptr() != rtop.data_ptr():
            top.copy_(rtop)
        if bottom is None:
            bottom = rbot
        elif bottom.data_ptr() != rbot.data_ptr():
            bottom.copy_(rbot)
        return top, bottom


LevelFn = Callable[[object, object, object], Sequence[object]]


def _call(fn, cur, top, bottom, outs):
    """Run a level (pair) function writing into `outs` when it accepts an
    `out=` argument (the GPU functions do: bands land in the Mallat buffer
    without a copy); otherwise copy its result in."""
    try:
        res = fn(cur, top, bottom, out=outs)
    except TypeError:
        res = fn(cur, top, bottom)
    return res


def _place(dst, src):
    if dst.data_ptr() != src.data_ptr():
        dst.copy_(src)


def forward_mallat_strips(level_fn: LevelFn, strip, levels: int, up: int, down: int,
                          exchange: Callable, out=None, pair_fn: Callable | None = None):
    """Strip-sharded forward pyramid. level_fn(strip, top, bottom[, out])
    returns the strip's four bands (LL, HL, LH, HH). pair_fn(strip, top,
    bottom[, out]), if given, runs levels 1 and 2 in one pass from 6*up /
    6*down halo rows and returns ([HL1, LH1, HH1], [LL2, HL2, LH2, HH2]).
    Functions that take `out=` write the detail bands straight into their
    quadrants of the strip-Mallat buffer. Works on torch tensors (CPU or
    CUDA). Returns the rank's strip-Mallat buffer."""
    import torch
    h0, w0 = strip.shape
    if out is None:
        out = torch.empty_like(strip)
    cur = strip
    first = 0
    if pair_fn is not None and levels >= 2:
        h, w = cur.shape
        check_strip(h, w, 3 * up, 3 * down)
        top, bottom = exchange(cur, 6 * up, 6 * down)
        h2, w2, h4, w4 = h // 2, w // 2, h // 4, w // 4
        ll2 = out[:h4, :w4] if levels == 2 else torch.empty((h4, w4), dtype=strip.dtype, device=strip.device)
        o1 = [out[:h2, w2:w], out[h2:h, :w2], out[h2:h, w2:w]]
        o2 = [ll2, out[:h4, w4:w2], out[h4:h2, :w4], out[h4:h2, w4:w2]]
        r1, r2 = _call(pair_fn, cur, top, bottom, (o1, o2))
        for d, s_ in zip(o1 + o2, list(r1) + list(r2)):
            _place(d, s_)
        cur, first = ll2, 2
    for lvl in range(first, levels):
        h, w = cur.shape
        check_strip(h, w, up, down)
        top, bottom = exchange(cur, 2 * up, 2 * down)
        h2, w2 = h // 2, w // 2
        last = lvl == levels - 1
        ll = out[:h2, :w2] if last else torch.empty((h2, w2), dtype=strip.dtype, device=strip.device)
        outs = [ll, out[:h2, w2:w], out[h2:h, :w2], out[h2:h, w2:w]]
        res = _call(level_fn, cur, top, bottom, outs)
        for d, s_ in zip(outs, res):
            _place(d, s_)
        cur = ll
    return out


def assemble_mallat(strips: Sequence, levels: int):
    """Global Mallat layout from the per-rank strip-Mallat buffers."""
    import torch
    n = len(strips)
    hs, W = strips[0].shape
    H = hs * n
    g = torch.empty((H, W), dtype=strips[0].dtype)
    w, h = W, H
    for lvl in range(levels):
        w2, h2 = w // 2, h // 2
        hl2 = (hs >> lvl) // 2  # band rows per rank at this level
        for r, s in enumerate(strips):
            s = s.cpu()
            hsl = hs >> lvl  # rank's level-input rows
            g[r * hl2:(r + 1) * hl2, w2:w] = s[:hl2, w2:w]
            g[h2 + r * hl2:h2 + (r + 1) * hl2, :w2] = s[hl2:hsl, :w2]
            g[h2 + r * hl2:h2 + (r + 1) * hl2, w2:w] = s[hl2:hsl, w2:w]
            if lvl == levels - 1:
                g[r * hl2:(r + 1) * hl2, :w2] = s[:hl2, :w2]
        w, h = w2, h2
    return g


def gpu_level_fn(plan, stream=None) -> LevelFn:
    """The product's level function: the fused sm_100a kernel with halo rows."""
    def fn(cur, top, bottom, out=None):
        return plan.forward_level_strip(cur, top, bottom, out=out, stream=stream)
    return fn


def gpu_forward_mallat(plan, strip, levels: int, exchange=None, out=None, scratch=None, stream=None):
    """The product's strip pyramid: the C++ driver (dwt2d_forward_mallat_strip)
    runs every level (levels 1+2 fused where the plan has the pair kernel)
    and calls back into `exchange` (e.g. a HaloExchange) for the halo rows."""
    ex = None if exchange is None else (lambda cur, tr, br, top, bottom: exchange(cur, tr, br, top, bottom))
    return plan.forward_mallat_strip(strip, levels, exchange=ex, out=out, scratch=scratch, stream=stream)


def gpu_pair_fn(plan, stream=None):
    """The product's fused level pair on a strip (None if the plan has none)."""
    if not plan.has_pair:
        return None

    def fn(cur, top, bottom, out=None):
        return plan.forward_pair_strip(cur, top, bottom, out=out, stream=stream)
    return fn


# ---------------------------------------------------------------------------
# Device-side sharded pyramid (the library's in-C++ multi-GPU driver,
# dwt2d_shard_* / dwt2d_forward_mallat_sharded): halo rows go straight into
# the ring neighbours' exchange windows over peer memory; no host callback,
# no collective library on the data path.

class Shard:
    """One rank of a row-strip sharded forward pyramid (dwt2d_shard) on the
    current CUDA device."""

    def __init__(self, plan, width: int, strip_height: int, levels: int, rank: int = 0, world: int = 1):
        import ctypes
        from . import native as N
        self._N = N
        self.plan = plan  # keeps the plan alive as long as the shard
        self.width, self.strip_height, self.levels = width, strip_height, levels
        self.rank, self.world = rank, world
        h = ctypes.c_void_p()
        N.check(N.lib.dwt2d_shard_create(plan._h, width, strip_height, levels, rank, world, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and getattr(self, "_N", None) is not None and self._N.lib is not None:
            self._N.lib.dwt2d_shard_destroy(h)
        self._h = None

    def export(self) -> bytes:
        """The exchange window's CUDA IPC handle (for ranks in other processes)."""
        import ctypes
        buf = ctypes.create_string_buffer(self._N.SHARD_HANDLE_BYTES)
        self._N.check(self._N.lib.dwt2d_shard_export(self._h, buf, len(buf)))
        return buf.raw

    def connect(self, prev: "Shard", nxt: "Shard") -> None:
        """Ring neighbours in this process (peer access is enabled)."""
        self._N.check(self._N.lib.dwt2d_shard_connect(self._h, prev._h, nxt._h))

    def connect_ipc(self, prev_handle: bytes, next_handle: bytes) -> None:
        """Ring neighbours in other processes, from their export() handles."""
        self._N.check(self._N.lib.dwt2d_shard_connect_ipc(self._h, prev_handle, next_handle))

    def forward_mallat(self, strip, out=None, stream=None, events=None):
        """Enqueue the whole strip pyramid (exchange included) on `stream`;
        returns the strip-Mallat buffer. events: None, or 1 + 4 * steps
        native.Event / None entries (dwt2d_shard_forward_mallat_ex)."""
        import ctypes
        import torch
        from .transform import _dev, _stream_handle
        H, W = strip.shape
        if out is None:
            out = torch.empty((H, W), dtype=torch.float32, device=strip.device)
        ptr, pitch = _dev(strip, "strip")
        optr, opitch = _dev(out, "out")
        if events is None:
            self._N.check(self._N.lib.dwt2d_shard_forward_mallat(self._h, ptr, pitch, optr, opitch,
                                                                 _stream_handle(stream)))
        else:
            if len(events) != 1 + 4 * self.info()["steps"]:
                raise ValueError("events needs 1 + 4 * steps entries")
            arr = (ctypes.c_void_p * len(events))(*[None if e is None else e.handle for e in events])
            self._N.check(self._N.lib.dwt2d_shard_forward_mallat_ex(self._h, ptr, pitch, optr, opitch, arr,
                                                                    _stream_handle(stream)))
        return out

    def info(self) -> dict:
        import ctypes
        steps, pair, hb = ctypes.c_int(), ctypes.c_int(), ctypes.c_size_t()
        self._N.check(self._N.lib.dwt2d_shard_info(self._h, ctypes.byref(steps), ctypes.byref(pair),
                                                   ctypes.byref(hb)))
        return {"steps": steps.value, "pair": bool(pair.value), "halo_bytes": hb.value}

    def status(self) -> int:
        """0, or the code of a halo wait that timed out (1: a neighbour never
        finished the previous pyramid, 2 / 3: the rows from the previous /
        next rank never arrived); readable after the trap (host memory).
        status_message() describes it."""
        import ctypes
        v = ctypes.c_int()
        self._N.check(self._N.lib.dwt2d_shard_status(self._h, ctypes.byref(v)))
        return v.value

    def status_message(self) -> str:
        return self._N.lib.dwt2d_last_error().decode() if self.status() else ""


def connect_ring(shards: Sequence["Shard"]) -> None:
    """Connect shards of one process into a ring (rank order)."""
    n = len(shards)
    if n > 1:
        for r, s in enumerate(shards):
            s.connect(shards[(r - 1) % n], shards[(r + 1) % n])


def dist_shard(plan, width: int, strip_height: int, levels: int, group=None) -> "Shard":
    """This process's shard of a ring spanning the torch.distributed group:
    creates it on the current device, exchanges the exchange-window handles
    (all_gather_object over the group) and maps the neighbours' windows."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    sh = Shard(plan, width, strip_height, levels, rank, world)
    if world > 1:
        handles = [None] * world
        dist.all_gather_object(handles, sh.export(), group=group)
        prev, nxt = ring_neighbours(rank, world)
        sh.connect_ipc(handles[prev], handles[nxt])
        dist.barrier(group)
    return sh


def forward_mallat_sharded(plan, strips: Sequence, levels: int, outs=None, streams=None):
    """Single-process multi-GPU pyramid (dwt2d_forward_mallat_sharded):
    strips[r] is rank r's strip on its device (devices may repeat: virtual
    ranks on one GPU). Returns the ranks' strip-Mallat buffers."""
    import ctypes
    import torch
    from . import native as N
    from .transform import _dev
    n = len(strips)
    H, W = strips[0].shape
    if outs is None:
        outs = [torch.empty((H, W), dtype=torch.float32, device=s.device) for s in strips]
    sp = [_dev(s, "strip") for s in strips]
    op = [_dev(o, "out") for o in outs]
    devs = (ctypes.c_int * n)(*[s.device.index if s.device.index is not None else 0 for s in strips])
    P = ctypes.c_void_p * n
    S = ctypes.c_size_t * n
    st = None
    if streams is not None:
        st = P(*[(s if isinstance(s, int) else s.cuda_stream) for s in streams])
    N.check(N.lib.dwt2d_forward_mallat_sharded(plan._h, n, devs, P(*[p for p, _ in sp]), S(*[q for _, q in sp]),
                                               W, H, levels, P(*[p for p, _ in op]), S(*[q for _, q in op]), st))
    return outs
