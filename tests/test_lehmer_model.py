"""Model of K6's blocked (Lehmer-style) remainder sequence -- the algorithm of
`blk_gcd_lehmer` in paper_1103_4697_b200/csrc/kernels_uni.cu, step for step, in Python ints.

The CUDA kernel runs the division-free Euclid of blk_gcd (kernels_uni.cu) in blocks: one warp
(the "leaf") takes the top T = 62 coefficients of X and Y into registers, runs as many steps
as those coefficients determine while it accumulates the 2x2 matrix of polynomials M with
(X_cur, Y_cur) = M (X_0, Y_0), and the whole CTA then applies M to the full polynomials (a
polynomial product of degree <= 30 by degree n, one barrier per block instead of one per
step).  Exactness is tracked by the lowest exact coefficient index lo of each window; a step
runs only when every coefficient it needs (its scalars, the new remainder's leading one) is
exact.  This file checks the model against a plain Euclid over F_p on random, structured and
degenerate inputs, so the block logic is proven before (and independently of) the kernel.
Pure test infrastructure: nothing in the product imports it.
"""

import random

import pytest

P = 1_000_000_007
T = 62        # window length (2 coefficients per lane, lanes 0..30 of one warp)
MD = 30       # max degree of the entries of M (one coefficient per lane, lanes 1..31)
ALL = -(1 << 20)  # "every index exact" (the window holds the whole polynomial)


def deg(a):
    d = len(a) - 1
    while d >= 0 and a[d] % P == 0:
        d -= 1
    return d


def gcd_deg_plain(a, b):
    a, b = [x % P for x in a], [x % P for x in b]
    da, db = deg(a), deg(b)
    while db >= 0:
        inv = pow(b[db], P - 2, P)
        while da >= db:
            q = a[da] * inv % P
            for i in range(db + 1):
                a[da - db + i] = (a[da - db + i] - q * b[i]) % P
            da = deg(a[:da])
        a, b, da, db = b, a, db, da
    return da


def poly_mul_add(m0, x, m1, y, n_out):
    """out[i] = sum_a m0[a] x[i-a] + m1[a] y[i-a], i in [0, n_out]."""
    out = [0] * (n_out + 1)
    for i in range(n_out + 1):
        s = 0
        for a in range(MD + 1):
            if 0 <= i - a < len(x):
                s += m0[a] * x[i - a]
            if 0 <= i - a < len(y):
                s += m1[a] * y[i - a]
        out[i] = s % P
    return out


def leaf(X, dx, Y, dy):
    """One block: returns (M, dx, dy, status, steps) with status 'ok' (both degrees exact),
    'done' (Y == 0 exactly: gcd = X), 'const' (deg Y = 0: gcd is a constant) or 'unknown'
    (the last remainder has no exact nonzero coefficient in the window)."""
    wx = [X[dx - j] if dx - j >= 0 else 0 for j in range(T)]
    wy = [Y[dy - j] if dy - j >= 0 else 0 for j in range(T)]
    lox = dx - T + 1 if dx >= T else ALL
    loy = dy - T + 1 if dy >= T else ALL
    mx = [[1] + [0] * MD, [0] * (MD + 1)]  # row X: (m00, m01)
    my = [[0] * (MD + 1), [1] + [0] * MD]  # row Y: (m10, m11)
    dmx = dmy = 0
    steps = 0

    def first_nonzero(w, dtop, lo):
        # returns z (shift) or None if no exact nonzero; the window entries for indices < 0 are 0
        for z in range(T):
            if dtop - z < max(lo, 0):
                break
            if w[z]:
                return z
        return None

    while True:
        if dy == 0:
            return (mx, my), dx, dy, "const", steps
        if dx == dy + 1:
            if dx - 1 < lox or dy - 1 < loy or dmy + 1 > MD:
                return (mx, my), dx, dy, "ok", steps
            b, a, x1, y1 = wy[0], wx[0], wx[1], wy[1]
            c1, c2, c3 = b * b % P, -b * a % P, -(b * x1 - a * y1) % P
            wr = [(c1 * (wx[j + 2] if j + 2 < T else 0) + c2 * (wy[j + 2] if j + 2 < T else 0)
                   + c3 * (wy[j + 1] if j + 1 < T else 0)) % P for j in range(T)]
            lr = max(lox, loy + 1)
            rows = [(c1 * mx[e][k] + c2 * (my[e][k - 1] if k else 0) + c3 * my[e][k]) % P
                    for e in range(2) for k in range(MD + 1)]
            mr = [rows[:MD + 1], rows[MD + 1:]]
            dmr = max(dmx, dmy + 1)
            steps += 1
            dt = dy - 1
            z = first_nonzero(wr, dt, lr)
            mx, my, dmx, dmy = my, mr, dmy, dmr
            wx, lox, dx = wy, loy, dy
            if z is None:
                if lr <= 0:
                    return (mx, my), dx, -1, "done", steps
                return (mx, my), dx, dt, "unknown", steps
            wy = wr[z:] + [0] * z
            loy, dy = lr, dt - z
        else:
            sh = dx - dy
            if dx < lox or dy < loy or dmy + sh > MD:
                return (mx, my), dx, dy, "ok", steps
            c, t = wy[0], -wx[0] % P
            wn = [(c * wx[j] + t * wy[j]) % P for j in range(T)]
            ln = max(lox, loy + sh)
            rows = [(c * mx[e][k] + t * (my[e][k - sh] if k >= sh else 0)) % P
                    for e in range(2) for k in range(MD + 1)]
            mx = [rows[:MD + 1], rows[MD + 1:]]
            dmx = max(dmx, dmy + sh)
            steps += 1
            z = first_nonzero(wn, dx, ln)
            if z is None:
                if ln <= 0:  # X == 0: gcd = Y; swap so the result sits in X
                    return (my, mx), dy, -1, "done", steps
                # X's degree unknown: hand back as (Y, X) so "unknown" always refers to Y
                return (my, mx), dy, dx - 1, "unknown", steps
            wx, lox, dx = wn[z:] + [0] * z, ln, dx - z
            if dx < dy:
                wx, wy, lox, loy, dx, dy = wy, wx, loy, lox, dy, dx
                mx, my, dmx, dmy = my, mx, dmy, dmx


def gcd_deg_lehmer(a, b):
    X, Y = [v % P for v in a], [v % P for v in b]
    dx, dy = deg(X), deg(Y)
    if dx < dy:
        X, Y, dx, dy = Y, X, dy, dx
    if dy < 0:
        return dx
    blocks = 0
    while True:
        blocks += 1
        if dy == 0:
            return 0
        if dx - dy > MD:
            # degree gap beyond M's reach: one direct elimination pass X <- c X - t x^sh Y
            c, t, sh = Y[dy], -X[dx] % P, dx - dy
            X = [(c * X[i] + (t * Y[i - sh] if 0 <= i - sh <= dy else 0)) % P for i in range(dx + 1)]
            dx = deg(X)
            if dx < 0:
                return dy
            if dx < dy:
                X, Y, dx, dy = Y, X, dy, dx
            continue
        (mx, my), ndx, ndy, st, steps = leaf(X, dx, Y, dy)
        assert steps > 0 or st == "const"
        if st == "const":
            return 0
        X2 = poly_mul_add(mx[0], X, mx[1], Y, ndx)
        Y2 = poly_mul_add(my[0], X, my[1], Y, max(ndy, 0)) if ndy >= 0 else [0]
        assert X2[ndx] != 0 and deg(X2) == ndx
        if st == "done":
            assert deg(Y2) == -1
            return ndx
        if st == "unknown":
            ndy = deg(Y2)
            if ndy < 0:
                return ndx
        else:
            assert deg(Y2) == ndy
        if ndy > ndx:
            X2, Y2, ndx, ndy = Y2, X2, ndy, ndx
        X, Y, dx, dy = X2, Y2, ndx, ndy


def rand_poly(rng, n):
    return [rng.randrange(P) for _ in range(n)] + [rng.randrange(1, P)]


def mul(a, b):
    out = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] = (out[i + j] + x * y) % P
    return out


def derivative(a):
    return [(i * a[i]) % P for i in range(1, len(a))] or [0]


CASES = []
_rng = random.Random(7)
for _n in (1, 2, 5, 40, 63, 64, 65, 130, 300):
    _f = rand_poly(_rng, _n)
    CASES.append(("sqfree-%d" % _n, _f, derivative(_f)))
for _n, _g in ((120, 3), (200, 40), (90, 70), (150, 1)):
    _G = rand_poly(_rng, _g)
    _f = mul(mul(_G, _G), rand_poly(_rng, _n))
    CASES.append(("square-%d-%d" % (_n, _g), _f, derivative(_f)))
for _n, _g in ((100, 10), (180, 100), (70, 69)):
    _G = rand_poly(_rng, _g)
    CASES.append(("common-%d-%d" % (_n, _g), mul(_G, rand_poly(_rng, _n)), mul(_G, rand_poly(_rng, _n - 7))))
# sparse / abnormal sequences: big degree drops, equal degrees, constants
CASES.append(("x^200+1 / x^200+x^3", [1] + [0] * 199 + [1], [0, 0, 0, 1] + [0] * 196 + [1]))
CASES.append(("x^150-1 / x^90-1", [P - 1] + [0] * 149 + [1], [P - 1] + [0] * 89 + [1]))
CASES.append(("x^300+x / 3x^299", [0, 1] + [0] * 298 + [1], [0] * 299 + [3]))
CASES.append(("y^16+g", [5, 7, 11] + [0] * 13 + [1], derivative([5, 7, 11] + [0] * 13 + [1])))
CASES.append(("gap-120", [3] + [0] * 119 + [1] + [2] * 30, [1] * 20 + [0] * 100 + [9] * 5))
CASES.append(("const", rand_poly(_rng, 80), [4]))
CASES.append(("equal-degree", rand_poly(_rng, 100), rand_poly(_rng, 100)))


@pytest.mark.parametrize("name,a,b", CASES, ids=[c[0] for c in CASES])
def test_lehmer_model_matches_euclid(name, a, b):
    assert gcd_deg_lehmer(a, b) == gcd_deg_plain(a, b)


def test_lehmer_model_random_degrees():
    rng = random.Random(11)
    for _ in range(25):
        g, u, w = rng.randrange(0, 40), rng.randrange(0, 120), rng.randrange(0, 120)
        G = rand_poly(rng, g)
        a, b = mul(G, rand_poly(rng, u)), mul(G, rand_poly(rng, w))
        assert gcd_deg_lehmer(a, b) == gcd_deg_plain(a, b)
