"""Synthetic curve workloads -- bit-identical to the oracle driver.

``dense(d, b, seed)``  every monomial x^i y^j with i + j <= d, drawn from one
                       ``std::mt19937_64(seed)`` in the order i = 0..d, j = 0..d-i;
                       magnitude built from 32-bit chunks, ``v == 0 -> 1``,
                       negative iff the next draw is odd.
``sheared(K, seed)``   f = g * prod_{k=1}^{K-1} g(x, y + k x + k), g = dense(6, 10, seed).

The generator is the workload definition used by ``bench.py`` and the tests;
``tests/test_curves.py`` checks it against ``oracle/_ref/refdriver gen`` (the reference side).
Polynomials are dicts ``{(deg_x, deg_y): int}``.
"""

from __future__ import annotations

_MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the C++11 64-bit Mersenne twister, default parameters)."""

    _N, _M = 312, 156
    _MATRIX_A = 0xB5026F5AA96619E9
    _UPPER, _LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        mt = [0] * self._N
        mt[0] = seed & _MASK64
        for i in range(1, self._N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK64
        self._mt = mt
        self._idx = self._N

    def _twist(self):
        mt, N, M = self._mt, self._N, self._M
        for i in range(N):
            x = (mt[i] & self._UPPER) | (mt[(i + 1) % N] & self._LOWER)
            xa = x >> 1
            if x & 1:
                xa ^= self._MATRIX_A
            mt[i] = mt[(i + M) % N] ^ xa
        self._idx = 0

    def __call__(self) -> int:
        if self._idx >= self._N:
            self._twist()
        y = self._mt[self._idx]
        self._idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64


def dense(d: int, b: int, seed: int) -> dict:
    rng = MT19937_64(seed)
    terms = {}
    for i in range(d + 1):
        for j in range(d - i + 1):
            v = 0
            done = 0
            while done < b:
                take = min(32, b - done)
                v = (v << take) + (rng() & ((1 << take) - 1))
                done += 32
            if v == 0:
                v = 1
            if rng() & 1:
                v = -v
            terms[(i, j)] = v
    return terms


def _bmul(a: dict, b: dict) -> dict:
    out: dict = {}
    for (ax, ay), ac in a.items():
        for (bx, by), bc in b.items():
            k = (ax + bx, ay + by)
            out[k] = out.get(k, 0) + ac * bc
    return {k: v for k, v in out.items() if v != 0}


def _badd(a: dict, b: dict) -> dict:
    out = dict(a)
    for k, v in b.items():
        out[k] = out.get(k, 0) + v
    return {k: v for k, v in out.items() if v != 0}


def shear(g: dict, k: int) -> dict:
    """g(x, y + k x + k)."""
    lin = {(0, 1): 1, (1, 0): k, (0, 0): k} if k else {(0, 1): 1}
    lin = {kk: v for kk, v in lin.items() if v != 0}
    dy = max(e[1] for e in g)
    out: dict = {}
    pw = {(0, 0): 1}
    for j in range(dy + 1):
        gj = {(ex, 0): c for (ex, ey), c in g.items() if ey == j}
        out = _badd(out, _bmul(gj, pw))
        pw = _bmul(pw, lin)
    return out


def sheared(K: int, seed: int) -> dict:
    g = dense(6, 10, seed)
    f = dict(g)
    for k in range(1, K):
        f = _bmul(f, shear(g, k))
    return f


def derive_y(f: dict) -> dict:
    return {(ex, ey - 1): c * ey for (ex, ey), c in f.items() if ey >= 1 and c * ey != 0}


def derive_x(f: dict) -> dict:
    return {(ex - 1, ey): c * ex for (ex, ey), c in f.items() if ex >= 1 and c * ex != 0}


# BASELINE.json configs -> (kind, a, b)
CONFIGS = {
    "d10_b10": ("dense", 10, 10),
    "d20_b64": ("dense", 20, 64),
    "d30_b128": ("dense", 30, 128),
    "sheared_k2": ("sheared", 2, 0),
    "sheared_k3": ("sheared", 3, 0),
    "d16_b1024": ("dense", 16, 1024),
}


def make(kind: str, a: int, b: int, seed: int) -> dict:
    if kind == "dense":
        return dense(a, b, seed)
    if kind == "sheared":
        return sheared(a, seed)
    raise ValueError(kind)
