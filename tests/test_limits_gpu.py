"""Inputs beyond the r1 size limits: the reference's entry points (elim.cpp:80-202) accept any
size, so the drop-in must too (no CTG_UNSUPPORTED).  Each case has an exact expected value
by construction, or (for the resultant at deg_y > 40) the CPU restatement / an exact closed
form, plus an evaluation-specialisation check over a 61-bit prime at random points."""

import random
import sys
import os

import pytest

import paper_1103_4697_b200 as P
from paper_1103_4697_b200 import curves

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import curvetop_oracle as O  # noqa: E402  (checker only)

pytestmark = pytest.mark.gpu

Q61 = 2**61 - 1


def _res_mod(a, b, q):
    """Sylvester resultant of dense univariate a (deg n), b (deg m) over F_q, formal degrees =
    actual (leading coefficients nonzero mod q): Euclid with res(A,B) = (-1)^{nm} lc(B)^{n-k} res(B,R)."""
    a = [c % q for c in a]
    b = [c % q for c in b]
    acc = 1
    while True:
        n, m = len(a) - 1, len(b) - 1
        if m == 0:
            return acc * pow(b[0], n, q) % q
        r = a[:]
        inv = pow(b[-1], q - 2, q)
        while len(r) - 1 >= m:
            t = r[-1] * inv % q
            s = len(r) - 1 - m
            for i in range(m + 1):
                r[s + i] = (r[s + i] - t * b[i]) % q
            r.pop()
        while r and r[-1] == 0:
            r.pop()
        if not r:
            return 0
        k = len(r) - 1
        acc = acc * pow(b[-1], n - k, q) % q
        if (n * m) & 1:
            acc = q - acc if acc else 0
        a, b = b, r


def _eval_rows(f, x0, q):
    n = max(ey for (_, ey) in f)
    rows = [0] * (n + 1)
    for (ex, ey), c in f.items():
        rows[ey] = (rows[ey] + c * pow(x0, ex, q)) % q
    return rows


def _upoly_eval(R, x0, q):
    acc = 0
    for c in reversed(R):
        acc = (acc * x0 + c) % q
    return acc


def _rand_curve(rng, ny, nx, bits):
    f = {(i, j): rng.randint(-(1 << bits), 1 << bits) for j in range(ny + 1) for i in range(nx + 1)}
    f[(0, ny)] = rng.choice((-3, -1, 1, 2, 5))  # constant leading y-coefficient: every x0 is a good point
    for i in range(1, nx + 1):
        f[(i, ny)] = 0
    return {k: v for k, v in f.items() if v}


def test_general_warp_kernel_against_restatement():
    """deg_y 45 / 43 (not a fast-path shape, above the thread kernel's 40): k_modres_warp,
    exact against the CPU restatement of elim.cpp:95-136."""
    rng = random.Random(45)
    p = _rand_curve(rng, 45, 1, 6)
    q = _rand_curve(rng, 43, 1, 6)
    assert P.resultant(p, q) == O.resultant(p, q, "y")


@pytest.mark.parametrize("n", [60, 150])
def test_superelliptic_beyond_128(n):
    """y^n + g(x): res(f, f_y) = n^n g^(n-1) exactly; n = 150 was CTG_UNSUPPORTED in r1."""
    rng = random.Random(n)
    g = [rng.randint(-9, 9) or 1 for _ in range(3)]
    f = {(i, 0): c for i, c in enumerate(g)}
    f[(0, n)] = 1
    want = [n ** n]
    for _ in range(n - 1):
        nxt = [0] * (len(want) + len(g) - 1)
        for i, a in enumerate(want):
            for j, b in enumerate(g):
                nxt[i + j] += a * b
        want = nxt
    assert P.resultant(f, curves.derive_y(f)) == want


def test_deg_y_150_specialisation():
    """A random deg_y 150 curve (warp kernel, 150 x 149 Sylvester shape): R(x0) mod q equals the
    F_q resultant of the specialised rows at random x0 (the leading y-coefficient is a constant,
    so every x0 specialises), and deg R <= the Bezout bound."""
    rng = random.Random(150)
    f = _rand_curve(rng, 150, 1, 8)
    fy = curves.derive_y(f)
    R = P.resultant(f, fy)
    assert 0 < len(R) - 1 <= 150 * 149
    for _ in range(3):
        x0 = rng.randrange(Q61)
        want = _res_mod(_eval_rows(f, x0, Q61), _eval_rows(fy, x0, Q61), Q61)
        assert _upoly_eval(R, x0, Q61) == want


def test_yun_beyond_shared_memory():
    """deg 6503 > the r1 cap of 6000 (K6 buffers in global memory):
    Yun((x-1)^2 (x+2) (x^6500 - 3)) = [((x+2)(x^6500-3), 1), (x-1, 2)] -- x^6500 - 3 is
    square-free and vanishes at neither 1 nor -2."""
    h = [-3] + [0] * 6499 + [1]
    a = O.u_mul([2, 1], h)
    Pp = O.u_mul(O.u_mul([-1, 1], [-1, 1]), a)
    unit, factors = P.yun_squarefree(Pp)
    assert unit == 1
    assert factors == [(a, 1), ([-1, 1], 2)]


def test_gcd_beyond_shared_memory():
    """deg 10501 (k_modgcd's five buffers exceed the shared-memory budget):
    gcd((x+3) g, (x-5) g) = g for primitive g with positive leading coefficient."""
    g = [1, -7] + [0] * 10498 + [1]
    assert P.gcd_univariate(O.u_mul([3, 1], g), O.u_mul([-5, 1], g)) == g


def test_gcd_bivariate_newton_beyond_shared_memory():
    """x-degree 900: the Newton interpolation needs N > 1,760 points (global scratch).
    gcd(h (y + x), h (y + x + 1)) = h for h = y + x^900 + 1 (primitive, lc_y = 1)."""
    h = {(0, 1): 1, (900, 0): 1, (0, 0): 1}
    f = O.b_mul(h, {(0, 1): 1, (1, 0): 1})
    g = O.b_mul(h, {(0, 1): 1, (1, 0): 1, (0, 0): 1})
    assert P.gcd_bivariate(f, g) == h


def _quad_curve(a, b):
    """f = y^2 + a(x) y + b(x): res(f, f_y) = 4 b - a^2 (res(g, f) = lc(g)^2 f(-a/2), n m even)."""
    f = {(0, 2): 1}
    for i, c in enumerate(a):
        if c:
            f[(i, 1)] = c
    for i, c in enumerate(b):
        if c:
            f[(i, 0)] = c
    return f


def test_result_degree_beyond_16383():
    """deg R = 20000 (N = 20480 > the shared-memory K4's 16384: global-memory NTT passes);
    exact: R = 4b - a^2 (numpy convolution, coefficients < 2^40)."""
    import numpy as np
    rng = np.random.default_rng(20000)
    a = rng.integers(-1023, 1024, size=10001).astype(np.int64)
    a[-1] = 7
    b = rng.integers(-1023, 1024, size=20001).astype(np.int64)
    want = (4 * b - np.convolve(a, a)).tolist()
    f = _quad_curve(a.tolist(), b.tolist())
    assert P.resultant(f, curves.derive_y(f)) == want


def test_prime_window_extension():
    """deg R = 80000 with ~10,000-bit coefficients: N = 81920 leaves ~200 primes p = cN + 1
    above 2^30, fewer than the bound needs -- the window extends below 2^30.  Checked exactly
    at the top and bottom coefficients and at random points mod a 61-bit prime."""
    rng = random.Random(80000)
    a = [rng.getrandbits(5000) * rng.choice((-1, 1)) for _ in range(40001)]
    b = [rng.randint(-1023, 1023) for _ in range(80001)]
    f = _quad_curve(a, b)
    R = P.resultant(f, curves.derive_y(f))
    assert len(R) == 80001
    assert R[-1] == 4 * b[-1] - a[-1] ** 2 and R[0] == 4 * b[0] - a[0] ** 2
    for _ in range(3):
        x0 = rng.randrange(Q61)
        av, bv = _upoly_eval(a, x0, Q61), _upoly_eval(b, x0, Q61)
        assert _upoly_eval(R, x0, Q61) == (4 * bv - av * av) % Q61


def test_crt_carry_chain_patterns():
    """Coefficients whose two's complement has long runs of zeros / ones across the fused CRT
    epilogue's segments (K5: tcgen05 GEMM + carry in the epilogue + k_crt_fixup): powers of two,
    2^k - 1, small values and zeros make the segment carries ripple (+1 through all-ones
    limbs, -1 through all-zeros limbs).  R = 4 b exactly for f = y^2 + b(x)."""
    vals = []
    for k in (31, 32, 63, 64, 65, 1000, 2047, 2048, 2049, 4000, 6143, 6144):
        vals += [2**k, -(2**k), 2**k - 1, -(2**k - 1), 2**k + 1, 3 * 2**k]
    vals += [0, 1, -1, 2, -5, 2**6000 - 2**3000, -(2**6000) + 2**64]
    b = vals + [1]
    f = {(0, 2): 1}
    for i, c in enumerate(b):
        if c:
            f[(i, 0)] = c
    R = P.resultant(f, curves.derive_y(f))
    want = [4 * c for c in b]
    while want and want[-1] == 0:
        want.pop()
    assert R == want
    # the same coefficients in a 16-curve batch (multi-tile rows of many curves)
    rng = random.Random(6144)
    pairs, wants = [], []
    for _ in range(16):
        bb = vals[:]
        rng.shuffle(bb)
        bb.append(7)
        g = {(0, 2): 1}
        g.update({(i, 0): c for i, c in enumerate(bb) if c})
        pairs.append((g, curves.derive_y(g)))
        wants.append([4 * c for c in bb])
    assert P.resultant_batch(pairs) == wants


@pytest.mark.parametrize("d", [41, 47, 48, 63, 64, 95, 100])
def test_multi_unit_warp_kernel_specialisation(d):
    """deg_y in (40, 127] with the derivative shape runs k_modres_mw (four units per warp, 8 lanes
    per unit, C = 6 / 8 / 12 / 16 coefficients per lane): R(x0) mod q == the F_q resultant of the
    specialised rows at random points, deg R <= d (d - 1), R(0) against the same check."""
    rng = random.Random(d)
    f = curves.dense(d, 8, 1000 + d)
    fy = curves.derive_y(f)
    R = P.resultant(f, fy)
    assert 0 < len(R) - 1 <= d * (d - 1)
    for x0 in [0, 1] + [rng.randrange(Q61) for _ in range(2)]:
        want = _res_mod(_eval_rows(f, x0, Q61), _eval_rows(fy, x0, Q61), Q61)
        assert _upoly_eval(R, x0, Q61) == want


def test_multi_unit_warp_kernel_staged_plan():
    """The staged plan API (K2 and K3 as separate stages, as bench.py times them) on a deg_y 50
    batch equals the one-call result: k_modres_mw reads K2's point values."""
    import torch
    pairs = [(f, curves.derive_y(f)) for f in (curves.dense(50, 8, s) for s in (1, 2, 3))]
    want = P.resultant_batch(pairs)
    plan = P.Plan(pairs)
    info = plan.info
    Pn, N, D, W = info["n_primes"], info["n_points"], info["n_coeffs"], info["out_limbs"] + 1
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    B = len(pairs)
    rows = torch.zeros((B, Pn, N), dtype=torch.int32, device="cuda")
    out = torch.zeros((B * D * W,), dtype=torch.int32, device="cuda")
    plan.upload(sh)
    for st_ in (1, 4, 5, 3):
        plan.stage(st_, 0, Pn, rows.data_ptr(), sh, curve_stride=Pn * N)
    plan.crt_batch(rows.data_ptr(), 0, D, out.data_ptr(), sh, curve_stride=Pn * N)
    torch.cuda.synchronize()
    plan.check(sh)
    host = out.cpu().numpy().view("uint32").reshape(B, D, W)
    assert [plan.decode(host[b]) for b in range(B)] == want


def test_yun_probe_beyond_small_primes():
    """Degree 33,000 (> 2^15): the square-freeness probe cannot use the primes below 2^15 and
    runs the blocked remainder sequence modulo the 31-bit primes, its buffers in global memory
    (four of 33,002 words); a random square-free input comes back as (sgn, [(P sgn, 1)])."""
    import random
    rng = random.Random(33)
    n = 33000
    poly = [rng.randrange(-1000, 1001) for _ in range(n)] + [rng.choice([-7, 7])]
    poly[0] = 1  # content 1
    sgn = -1 if poly[-1] < 0 else 1
    assert P.yun_squarefree(poly) == (sgn, [([sgn * c for c in poly], 1)])
