"""Synthetic inputs, bit-identical to the reference's generator.

random_image (reference random.hpp:13-37): a 64-bit LCG with Knuth's MMIX
constants, one draw per sample in row-major order, sample = (s >> 11) * 2^-53
cast to float32. Generated on the device with affine jump-ahead: the state
after k draws is A_k * seed + C_k (mod 2^64), so any row band (one GPU's
strip of a sharded image) is produced independently and bit-identically.
int64 tensor arithmetic wraps modulo 2^64 exactly like uint64.
"""
from __future__ import annotations

MUL = 6364136223846793005
ADD = 1442695040888963407
M64 = (1 << 64) - 1


def _jump(k: int) -> tuple[int, int]:
    """(A, C) with state_{n+k} = A * state_n + C (mod 2^64)."""
    a, c, ma, mc = 1, 0, MUL, ADD
    while k:
        if k & 1:
            a, c = (ma * a) & M64, (ma * c + mc) & M64
        ma, mc = (ma * ma) & M64, (ma * mc + mc) & M64
        k >>= 1
    return a, c


def _s64(v: int) -> int:
    v &= M64
    return v - (1 << 64) if v >= (1 << 63) else v


def random_image(width: int, height: int, seed: int = 1, *, row0: int = 0, rows: int | None = None,
                 device="cuda"):
    """Rows [row0, row0 + rows) of random_image<float>(width, height, seed)
    as a float32 tensor on `device`."""
    import torch
    rows = height - row0 if rows is None else rows
    dev = torch.device(device)
    # per-column affine maps for draws 1..width within a row
    ak, ck = [], []
    a, c = 1, 0
    for _ in range(width):
        a, c = (MUL * a) & M64, (MUL * c + ADD) & M64
        ak.append(_s64(a))
        ck.append(_s64(c))
    A = torch.tensor(ak, dtype=torch.int64, device=dev)
    C = torch.tensor(ck, dtype=torch.int64, device=dev)
    # state before the first draw of each row
    ja, jc = _jump(row0 * width)
    s = (ja * seed + jc) & M64
    ra, rc = _jump(width)
    starts = []
    for _ in range(rows):
        starts.append(_s64(s))
        s = (ra * s + rc) & M64
    S = torch.tensor(starts, dtype=torch.int64, device=dev)
    out = torch.empty((rows, width), dtype=torch.float32, device=dev)
    step = max(1, (1 << 26) // max(1, width))
    for r0 in range(0, rows, step):
        st = S[r0:r0 + step, None] * A[None, :] + C[None, :]
        top = (st >> 11) & ((1 << 53) - 1)
        out[r0:r0 + step] = (top.to(torch.float64) * 2.0 ** -53).to(torch.float32)
    return out
