"""K6's blocked (Lehmer-style) remainder sequence on the GPU (lehmer.cuh, through the
ctg_modp_gcd_degree hook) against a plain Euclid over F_p in Python ints and against the
one-pass-per-step kernel (blk_gcd).  The block logic itself is modelled in test_lehmer_model.py;
here the kernel is checked on the same kinds of inputs: square-free (the probe's normal case),
squares and common factors (nonzero gcd degree), sparse inputs with large degree drops and gaps
beyond the matrix's reach, constants, and degrees past the shared-memory budget (global buffers).
"""

import os
import random

import pytest

import paper_1103_4697_b200 as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def p():
    return P.uni_prime(0, device=0)


def deg(a, p):
    d = len(a) - 1
    while d >= 0 and a[d] % p == 0:
        d -= 1
    return d


def gcd_deg(a, b, p):
    a, b = [x % p for x in a], [x % p for x in b]
    da, db = deg(a, p), deg(b, p)
    if da < db:
        a, b, da, db = b, a, db, da
    while db >= 0:
        inv = pow(b[db], p - 2, p)
        while da >= db:
            q = a[da] * inv % p
            if q:
                for i in range(db + 1):
                    a[da - db + i] = (a[da - db + i] - q * b[i]) % p
            da = deg(a[:da], p)
        a, b, da, db = b, a, db, da
    return da


def rand_poly(rng, n, p):
    return [rng.randrange(p) for _ in range(n)] + [rng.randrange(1, p)]


def mul(a, b, p):
    out = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        if x:
            for j, y in enumerate(b):
                out[i + j] = (out[i + j] + x * y) % p
    return out


def derivative(a, p):
    return [(i * a[i]) % p for i in range(1, len(a))] or [0]


def cases(p):
    rng = random.Random(5)
    out = []
    for n in (1, 2, 3, 31, 32, 33, 63, 64, 65, 66, 127, 128, 129, 300, 870):
        f = rand_poly(rng, n, p)
        out.append((f"sqfree-{n}", f, derivative(f, p)))
    for n, g in ((120, 3), (200, 40), (90, 70), (150, 1), (400, 100)):
        G = rand_poly(rng, g, p)
        f = mul(mul(G, G, p), rand_poly(rng, n, p), p)
        out.append((f"square-{n}-{g}", f, derivative(f, p)))
    for n, g in ((100, 10), (180, 100), (70, 69), (500, 33)):
        G = rand_poly(rng, g, p)
        out.append((f"common-{n}-{g}", mul(G, rand_poly(rng, n, p), p), mul(G, rand_poly(rng, n - 7, p), p)))
    out.append(("x^200+1|x^200+x^3", [1] + [0] * 199 + [1], [0, 0, 0, 1] + [0] * 196 + [1]))
    out.append(("x^150-1|x^90-1", [p - 1] + [0] * 149 + [1], [p - 1] + [0] * 89 + [1]))
    out.append(("x^300+x|3x^299", [0, 1] + [0] * 298 + [1], [0] * 299 + [3]))
    y16 = [5, 7, 11] + [0] * 13 + [1]
    out.append(("y^16+g", y16, derivative(y16, p)))
    out.append(("gap-120", [3] + [0] * 119 + [1] + [2] * 30, [1] * 20 + [0] * 100 + [9] * 5))
    out.append(("const", rand_poly(rng, 80, p), [4]))
    out.append(("zero", rand_poly(rng, 80, p), [0]))
    out.append(("both-zero", [0, 0], [0]))
    out.append(("equal-degree", rand_poly(rng, 100, p), rand_poly(rng, 100, p)))
    # runs of zero coefficients in the middle: remainders whose exact window vanishes
    sparse = [rng.randrange(1, p) if (i % 37) < 3 else 0 for i in range(400)] + [1]
    out.append(("sparse-runs", sparse, derivative(sparse, p)))
    lac = [0] * 1001
    for e in (0, 1, 64, 129, 500, 1000):
        lac[e] = rng.randrange(1, p)
    out.append(("lacunary", lac, derivative(lac, p)))
    return out


_NAMES = [c[0] for c in cases(1_000_000_007)]


@pytest.mark.parametrize("idx", range(len(_NAMES)), ids=_NAMES)
def test_gcd_degree_matches_euclid(p, idx):
    name, a, b = cases(p)[idx]
    want = gcd_deg(a, b, p)
    for method in (0, 1):
        got = P.modp_gcd_degree(a, b, 0, method, device=0)
        assert got["prime"] == p
        assert got["deg"] == want, (name, method, got, want)


@pytest.mark.parametrize("idx", range(len(_NAMES)), ids=_NAMES)
def test_gcd_degree_small_prime(idx):
    """The probe's 32-bit arithmetic (lehmer::SmallA) modulo the probe primes (< 2^15)."""
    for k in (0, 2):
        q = P.uni_prime(k, device=0, method=2)
        assert 1 << 14 < q < 1 << 15
        name, a, b = cases(q)[idx]
        got = P.modp_gcd_degree(a, b, k, 2, device=0)
        assert got["prime"] == q
        assert got["deg"] == gcd_deg(a, b, q), (name, k, got)


@pytest.mark.parametrize("n,g", [(2000, 0), (6000, 25), (13000, 7)])
def test_gcd_degree_large(p, n, g):
    """Beyond the shared-memory budget at 13,000 (four buffers of 52 KB): global buffers."""
    rng = random.Random(n)
    G = rand_poly(rng, g, p)
    a = mul(G, rand_poly(rng, n, p), p)
    b = mul(G, rand_poly(rng, n - 3, p), p)
    r0 = P.modp_gcd_degree(a, b, 0, 0, device=0)
    r1 = P.modp_gcd_degree(a, b, 0, 1, device=0)
    assert r0["deg"] == r1["deg"] == g  # coprime cofactors with overwhelming probability
    print(f"n={n}: blocked {r0['ms']:.3f} ms, one pass per step {r1['ms']:.3f} ms")
    if n < 1 << 14:
        q = P.uni_prime(0, device=0, method=2)
        G = rand_poly(rng, g, q)
        a = mul(G, rand_poly(rng, n, q), q)
        b = mul(G, rand_poly(rng, n - 3, q), q)
        assert P.modp_gcd_degree(a, b, 0, 2, device=0)["deg"] == g


def test_gcd_degree_other_primes():
    rng = random.Random(3)
    for k in (1, 2, 5):
        p = P.uni_prime(k, device=0)
        G = rand_poly(rng, 12, p)
        f = mul(mul(G, G, p), rand_poly(rng, 200, p), p)
        assert P.modp_gcd_degree(f, derivative(f, p), k, 0, device=0)["deg"] == gcd_deg(f, derivative(f, p), p)


def test_gcd_degree_random_stress():
    """Randomised mix of the structures above (planted common factors, sparse supports with long
    zero runs, equal and far-apart degrees) in both arithmetics, against Python's Euclid."""
    rng = random.Random(2024)
    q = P.uni_prime(1, device=0, method=2)
    p = P.uni_prime(0, device=0)
    for it in range(int(os.environ.get("CTG_STRESS_N", "120"))):
        mod, method, k = (p, 0, 0) if it % 2 == 0 else (q, 2, 1)
        g = rng.choice([0, 0, 1, 3, 17, 40, 75])
        G = rand_poly(rng, g, mod)

        def cofactor(n):
            if rng.random() < 0.3:  # sparse: a few nonzero coefficients, long zero runs
                c = [0] * n + [rng.randrange(1, mod)]
                for _ in range(rng.randrange(1, 5)):
                    c[rng.randrange(0, n + 1)] = rng.randrange(1, mod)
                return c
            return rand_poly(rng, n, mod)
        a = mul(G, cofactor(rng.randrange(1, 300)), mod)
        b = mul(G, cofactor(rng.randrange(0, 300)), mod) if rng.random() < 0.8 else derivative(a, mod)
        got = P.modp_gcd_degree(a, b, k, method, device=0)
        assert got["deg"] == gcd_deg(a, b, mod), (it, method, len(a) - 1, len(b) - 1, got)
