"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference DWT path.

This module is the CPU oracle the parity tests check the CUDA product
against. It is never imported by the product package; only tests/,
``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` leg may use it.

It restates, in float64 numpy, the reference algorithm for the hot path:

* Laurent polynomials over exact rationals (``fractions.Fraction``) or reals
  — reference ``laurent.hpp:14-82``, ``coeff.hpp:13-46``; key (m, n) reads
  component sample (x + m, y + n).
* the 4x4 lifting/spatial/polyconvolution matrices and the five scheme
  builders, inverse lifting and the constant-split optimizer
  — ``src/scheme.cpp:15-378``.
* the naive interpreter the reference's own unit tests use as their oracle
  (``tests/test_executor.cpp:21-47``): pre-scale, apply each fused group's
  composed matrix with the component-grid extension (``image.hpp:14-26``),
  post-scale.
* the LCG image generator (``random.hpp:13-37``) and polyphase split/merge
  (``image.hpp:73-113``), and the Mallat multi-level loop.

Parity is pinned: tests/test_oracle.py checks this module against the
compiled reference (``oracle/_ref``) and against the committed golden
fixtures in tests/golden/ (generated from the reference by
scripts/make_golden.py).
"""
from __future__ import annotations

from fractions import Fraction
from typing import Dict, List, Tuple

import numpy as np

Key = Tuple[int, int]
Poly = Dict[Key, object]  # coefficient: Fraction (exact) or float (real)

# ---------------------------------------------------------------------------
# coefficients and polynomials (coeff.cpp, laurent.cpp)


def _add(a, b):
    if isinstance(a, Fraction) and isinstance(b, Fraction):
        return a + b
    return float(a) + float(b)


def _mul(a, b):
    if isinstance(a, Fraction) and isinstance(b, Fraction):
        return a * b
    return float(a) * float(b)


def _is_zero(c) -> bool:
    return c == 0


def p_norm(p: Poly) -> Poly:
    return {k: c for k, c in sorted(p.items()) if not _is_zero(c)}


def p_add(a: Poly, b: Poly) -> Poly:
    out = dict(a)
    for k, c in b.items():
        out[k] = _add(out[k], c) if k in out else c
    return p_norm(out)


def p_neg(a: Poly) -> Poly:
    return {k: (-c) for k, c in a.items()}


def p_mul(a: Poly, b: Poly) -> Poly:
    out: Dict[Key, object] = {}
    for ka, ca in a.items():
        for kb, cb in b.items():
            k = (ka[0] + kb[0], ka[1] + kb[1])
            v = _mul(ca, cb)
            out[k] = _add(out[k], v) if k in out else v
    return p_norm(out)


def p_transpose(a: Poly) -> Poly:
    return p_norm({(k[1], k[0]): c for k, c in a.items()})


def p_embed(a: Poly, vertical: bool) -> Poly:
    """laurent.cpp:120-126 — univariate-in-m polynomial onto an axis."""
    assert all(k[1] == 0 for k in a), "not univariate"
    return p_transpose(a) if vertical else dict(a)


ONE: Poly = {(0, 0): Fraction(1)}


def p_const(c) -> Poly:
    return p_norm({(0, 0): c})


def p_split_constant(a: Poly) -> Tuple[Poly, Poly]:
    """laurent.cpp:128-131."""
    c = p_const(a.get((0, 0), Fraction(0)))
    return c, p_add(a, p_neg(c))


def p_is_one(a: Poly) -> bool:
    return len(a) == 1 and (0, 0) in a and a[(0, 0)] == 1


# ---------------------------------------------------------------------------
# 4x4 matrices (polymatrix.cpp) — list of 16 polys, row-major, comps ee oe eo oo


def m_identity(n=4):
    return [dict(ONE) if r == c else {} for r in range(n) for c in range(n)]


def m_mul(a, b, n=4):
    out = []
    for r in range(n):
        for c in range(n):
            acc: Poly = {}
            for k in range(n):
                acc = p_add(acc, p_mul(a[r * n + k], b[k * n + c]))
            out.append(acc)
    return out


def lift4(r1, c1, r2, c2, p):
    """scheme.cpp:15-20."""
    m = m_identity()
    m[r1 * 4 + c1] = p
    m[r2 * 4 + c2] = p
    return m


def predict_h(p):  # scheme.cpp:108-110
    return lift4(1, 0, 3, 2, p_embed(p, False))


def predict_v(p):  # scheme.cpp:112-114
    return lift4(2, 0, 3, 1, p_embed(p, True))


def update_h(u):  # scheme.cpp:116-118
    return lift4(0, 1, 2, 3, p_embed(u, False))


def update_v(u):  # scheme.cpp:120-122
    return lift4(0, 2, 1, 3, p_embed(u, True))


def spatial_predict(p):  # scheme.cpp:128-138, T[P]
    ph = p_embed(p, False)
    pv = p_transpose(ph)
    m = m_identity()
    m[1 * 4 + 0] = ph
    m[2 * 4 + 0] = pv
    m[3 * 4 + 0] = p_mul(ph, pv)
    m[3 * 4 + 1] = pv
    m[3 * 4 + 2] = ph
    return m


def spatial_update(u):  # scheme.cpp:140-150, S[U]
    uh = p_embed(u, False)
    uv = p_transpose(uh)
    m = m_identity()
    m[0 * 4 + 1] = uh
    m[0 * 4 + 2] = uv
    m[0 * 4 + 3] = p_mul(uh, uv)
    m[1 * 4 + 3] = uv
    m[2 * 4 + 3] = uh
    return m


def polyconv_matrix(p, u):  # scheme.cpp:152-177, N[P,U]
    ph, uh = p_embed(p, False), p_embed(u, False)
    v = p_add(p_mul(ph, uh), ONE)
    pt, ut, vt = p_transpose(ph), p_transpose(uh), p_transpose(v)
    rows = [
        [p_mul(vt, v), p_mul(vt, uh), p_mul(ut, v), p_mul(ut, uh)],
        [p_mul(vt, ph), vt, p_mul(ut, ph), ut],
        [p_mul(pt, v), p_mul(pt, uh), v, uh],
        [p_mul(pt, ph), pt, ph, dict(ONE)],
    ]
    return [rows[r][c] for r in range(4) for c in range(4)]


# ---------------------------------------------------------------------------
# wavelets (wavelet.cpp:16-59)

ALPHA = -1.586134342059924
BETA = -0.052980118572961
GAMMA = 0.882911075530934
DELTA = 0.443506852043971
ZETA = 1.149604398860241


def _uni(taps):
    return p_norm({(k, 0): c for k, c in taps})


F = Fraction
WAVELETS = {
    "cdf53": ([(_uni([(0, F(-1, 2)), (1, F(-1, 2))]), _uni([(-1, F(1, 4)), (0, F(1, 4))]))], 1.0),
    "cdf97": ([(_uni([(0, ALPHA), (1, ALPHA)]), _uni([(-1, BETA), (0, BETA)])),
               (_uni([(0, GAMMA), (1, GAMMA)]), _uni([(-1, DELTA), (0, DELTA)]))], ZETA),
    "dd137": ([(_uni([(-1, F(1, 16)), (0, F(-9, 16)), (1, F(-9, 16)), (2, F(1, 16))]),
                _uni([(-2, F(-1, 32)), (-1, F(9, 32)), (0, F(9, 32)), (1, F(-1, 32))]))], 1.0),
}

SCHEMES = ["separable-convolution", "separable-lifting", "nonseparable-convolution",
           "nonseparable-polyconvolution", "nonseparable-lifting"]


def _scale_diag(zeta):  # scheme.cpp:22-25
    return [zeta * zeta, 1.0, 1.0, 1.0 / (zeta * zeta)]


class Scheme:
    """scheme.hpp: steps = list of fused groups; each group = list of factors,
    factors[0] is leftmost (applied last)."""

    def __init__(self, kind, steps, pre=None, post=None):
        self.kind = kind
        self.steps = steps
        self.pre = pre or [1.0] * 4
        self.post = post or [1.0] * 4

    def composed(self, i):
        acc = self.steps[i][0]
        for f in self.steps[i][1:]:
            acc = m_mul(acc, f)
        return acc


def _conv_mats(pairs):
    nh, nv = m_identity(), m_identity()
    for p, u in pairs:
        nh = m_mul(update_h(u), m_mul(predict_h(p), nh))
        nv = m_mul(update_v(u), m_mul(predict_v(p), nv))
    return nh, nv


def build_scheme(kind: str, wavelet: str) -> Scheme:
    """scheme.cpp:191-258."""
    pairs, zeta = WAVELETS[wavelet]
    post = _scale_diag(zeta)
    if kind == "separable-convolution":
        nh, nv = _conv_mats(pairs)
        steps = [[nh], [nv]]
    elif kind == "separable-lifting":
        steps = []
        for p, u in pairs:
            steps += [[predict_h(p)], [predict_v(p)], [update_h(u)], [update_v(u)]]
    elif kind == "nonseparable-convolution":
        nh, nv = _conv_mats(pairs)
        steps = [[m_mul(nv, nh)]]
    elif kind == "nonseparable-polyconvolution":
        steps = [[polyconv_matrix(p, u)] for p, u in pairs]
    elif kind == "nonseparable-lifting":
        steps = []
        for p, u in pairs:
            steps += [[spatial_predict(p)], [spatial_update(u)]]
    else:
        raise ValueError(kind)
    return Scheme(kind, steps, post=post)


def build_inverse_lifting(wavelet: str) -> Scheme:
    """scheme.cpp:260-277."""
    pairs, zeta = WAVELETS[wavelet]
    steps = []
    for p, u in reversed(pairs):
        steps += [[update_v(p_neg(u))], [update_h(p_neg(u))],
                  [predict_v(p_neg(p))], [predict_h(p_neg(p))]]
    d = _scale_diag(zeta)
    return Scheme("inverse-lifting", steps, pre=[1.0 / x for x in d])


def optimize_constant_split(s: Scheme, wavelet: str) -> Scheme:
    """scheme.cpp:279-378 — same step count, each group's product unchanged."""
    pairs, _ = WAVELETS[wavelet]
    out = Scheme(s.kind, [], pre=s.pre, post=s.post)
    if s.kind == "separable-lifting":
        out.steps = s.steps
        return out
    if s.kind == "nonseparable-lifting":
        for p, u in pairs:
            p0, p1 = p_split_constant(p)
            g = [spatial_predict(p1)]
            if p0:
                g += [predict_v(p0), predict_h(p0)]
            out.steps.append(g)
            u0, u1 = p_split_constant(u)
            g = [spatial_update(u1)]
            if u0:
                g += [update_v(u0), update_h(u0)]
            out.steps.append(g)
        return out
    if s.kind == "nonseparable-polyconvolution":
        for p, u in pairs:
            p0, p1 = p_split_constant(p)
            u0, u1 = p_split_constant(u)
            g = []
            if u0:
                g += [update_v(u0), update_h(u0)]
            g.append(polyconv_matrix(p1, u1))
            if p0:
                g += [predict_v(p0), predict_h(p0)]
            out.steps.append(g)
        return out
    pf0, pf1 = p_split_constant(pairs[0][0])
    ul0, ul1 = p_split_constant(pairs[-1][1])
    mh, mv = m_identity(), m_identity()
    for k, (p, u) in enumerate(pairs):
        pp = pf1 if k == 0 else p
        uu = ul1 if k + 1 == len(pairs) else u
        mh = m_mul(update_h(uu), m_mul(predict_h(pp), mh))
        mv = m_mul(update_v(uu), m_mul(predict_v(pp), mv))
    if s.kind == "separable-convolution":
        h = ([update_h(ul0)] if ul0 else []) + [mh] + ([predict_h(pf0)] if pf0 else [])
        v = ([update_v(ul0)] if ul0 else []) + [mv] + ([predict_v(pf0)] if pf0 else [])
        out.steps = [h, v]
        return out
    g = ([update_v(ul0), update_h(ul0)] if ul0 else []) + [m_mul(mv, mh)]
    g += [predict_v(pf0), predict_h(pf0)] if pf0 else []
    out.steps = [g]
    return out


def make(wavelet: str, scheme: str, optimized: bool = False) -> Scheme:
    if scheme == "inverse-lifting":
        return build_inverse_lifting(wavelet)
    s = build_scheme(scheme, wavelet)
    return optimize_constant_split(s, wavelet) if optimized else s


def count_operations(s: Scheme) -> int:
    """scheme.cpp:382-393."""
    ops = 0
    for g in s.steps:
        for m in g:
            for r in range(4):
                for c in range(4):
                    p = m[r * 4 + c]
                    ops += len(p_add(p, p_neg(ONE))) if r == c else len(p)
    return ops


# ---------------------------------------------------------------------------
# images (image.hpp, random.hpp)


def extend_index(i: int, n: int, symmetric: bool) -> int:
    """image.hpp:14-26."""
    if n <= 0:
        raise ValueError("extend_index: empty axis")
    if 0 <= i < n:
        return i
    if not symmetric:
        return i % n
    if n == 1:
        return 0
    period = 2 * n - 2
    r = i % period
    return r if r < n else period - r


_LCG_A = 6364136223846793005
_LCG_C = 1442695040888963407
_M64 = (1 << 64) - 1


def lcg_draws(count: int, seed: int, start: int = 0) -> np.ndarray:
    """random.hpp:13-28: state <- a*state + c (mod 2^64); unit = (s>>11)*2^-53.
    Vectorised with affine jump-ahead: state_k = A_k*seed + C_k."""
    # jump to `start`
    a, c = 1, 0
    ma, mc, e = _LCG_A, _LCG_C, start
    while e:
        if e & 1:
            a, c = (ma * a) & _M64, (ma * c + mc) & _M64
        ma, mc = (ma * ma) & _M64, (ma * mc + mc) & _M64
        e >>= 1
    s0 = (a * seed + c) & _M64
    # states s0*A^k + C_k for k = 1..count via uint64 wrap-around arithmetic
    out = np.empty(count, dtype=np.uint64)
    block = 1 << 12
    # per-offset multipliers within a block
    ak = np.empty(block, dtype=np.uint64)
    ck = np.empty(block, dtype=np.uint64)
    ca, cc = 1, 0
    for k in range(block):
        ca, cc = (_LCG_A * ca) & _M64, (_LCG_A * cc + _LCG_C) & _M64
        ak[k], ck[k] = ca, cc
    base = s0
    with np.errstate(over="ignore"):
        for b0 in range(0, count, block):
            n = min(block, count - b0)
            out[b0:b0 + n] = ak[:n] * np.uint64(base) + ck[:n]
            base = int(out[b0 + n - 1])
    return (out >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def random_image(w: int, h: int, seed: int, dtype=np.float32) -> np.ndarray:
    """random.hpp:31-37 — double draw then cast to T (round to nearest)."""
    return lcg_draws(w * h, seed).reshape(h, w).astype(dtype)


def split(img):
    """image.hpp:73-94."""
    H, W = img.shape
    if H <= 0 or W <= 0 or H % 2 or W % 2:
        raise ValueError("polyphase_split: empty or odd image")
    return [np.ascontiguousarray(img[(j >> 1)::2, (j & 1)::2]) for j in range(4)]


def merge(planes):
    """image.hpp:96-113."""
    h2, w2 = planes[0].shape
    img = np.empty((2 * h2, 2 * w2), dtype=planes[0].dtype)
    for j in range(4):
        img[(j >> 1)::2, (j & 1)::2] = planes[j]
    return img


# ---------------------------------------------------------------------------
# executor semantics (test_executor.cpp:21-47 naive interpreter; extension
# applied per composed tap on the component grid as executor.hpp:159-167)


def _shifted(plane: np.ndarray, m: int, n: int, symmetric: bool) -> np.ndarray:
    """Array whose (y, x) holds plane[ext(y+n), ext(x+m)]."""
    h2, w2 = plane.shape
    ys = np.array([extend_index(y + n, h2, symmetric) for y in range(h2)])
    xs = np.array([extend_index(x + m, w2, symmetric) for x in range(w2)])
    return plane[np.ix_(ys, xs)]


def _coef(c) -> float:
    return float(c)


def apply_matrix(mat, planes, symmetric=False):
    out = []
    for r in range(4):
        acc = np.zeros_like(planes[0], dtype=np.float64)
        for j in range(4):
            for (m, n), c in mat[r * 4 + j].items():
                acc += _coef(c) * _shifted(planes[j], m, n, symmetric)
        out.append(acc)
    return out


def run(s: Scheme, planes, symmetric=False):
    """Float64 transform of four component planes through every step."""
    cur = [np.asarray(p, dtype=np.float64) * s.pre[j] for j, p in enumerate(planes)]
    for i in range(len(s.steps)):
        cur = apply_matrix(s.composed(i), cur, symmetric)
    return [c * s.post[r] for r, c in enumerate(cur)]


def transform(wavelet, scheme, planes, optimized=False, symmetric=False):
    return run(make(wavelet, scheme, optimized), planes, symmetric)


def pyramid(wavelet, scheme, img, levels, optimized=False, symmetric=False):
    """Mallat loop in float64; Mallat layout output."""
    s = make(wavelet, scheme, optimized)
    out = np.array(img, dtype=np.float64)
    H, W = out.shape
    w, h = W, H
    for _ in range(levels):
        res = run(s, split(out[:h, :w]), symmetric)
        w2, h2 = w // 2, h // 2
        out[:h2, :w2] = res[0]
        out[:h2, w2:w] = res[1]
        out[h2:h, :w2] = res[2]
        out[h2:h, w2:w] = res[3]
        w, h = w2, h2
    return out


def level_errors(got: np.ndarray, truth: np.ndarray, img: np.ndarray, levels: int):
    """SURVEY §8(c) parity metric: per level l, max |got - truth| over the
    four bands written at that level, divided by the peak |input| of level l
    (level 1: the image; level l: the float64 LL_{l-1})."""
    H, W = truth.shape
    errs = []
    w, h = W, H
    ll = np.asarray(img, dtype=np.float64)
    for lev in range(levels):
        peak = float(np.max(np.abs(ll))) or 1.0
        w2, h2 = w // 2, h // 2
        last = lev == levels - 1
        regions = [(slice(0, h2), slice(w2, w)), (slice(h2, h), slice(0, w2)),
                   (slice(h2, h), slice(w2, w))]
        if last:
            regions.append((slice(0, h2), slice(0, w2)))
        e = max(float(np.max(np.abs(got[r].astype(np.float64) - truth[r]))) for r in regions)
        errs.append(e / peak)
        ll = truth[:h2, :w2]
        w, h = w2, h2
    return errs
