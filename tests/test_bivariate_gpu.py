"""SURVEY.md §8(f) ranks 1-2 on the GPU: gcd_bivariate (elim.cpp:178-202) and the Teissier
resultant Q = res(f_x / h, f_y / h) with Yun(Q) (CurveContext::resultant_q, lift.cpp:76-101).

Expected values: the reference itself (tests/golden/bivariate_gcd.jsonl, teissier.jsonl made
by oracle/make_golden.py through oracle/_ref/refdriver).  Bit-exact equality required.
"""

import pytest

import curvetop_oracle as O
import paper_1103_4697_b200 as P
from golden_io import dec_bipoly, dec_sqf, dec_upoly, load
from paper_1103_4697_b200 import curves

pytestmark = pytest.mark.gpu


def _sqf(res):
    unit, factors = res
    return unit, [(list(f), m) for f, m in factors]


def test_gcd_bivariate_against_reference():
    rows = load("bivariate_gcd.jsonl")
    assert len(rows) > 80
    n_coprime = n_shared = 0
    for r in rows:
        f, g = (dec_bipoly(a) for a in r["args"])
        if "error" in r:
            with pytest.raises(P.PreconditionError):
                P.gcd_bivariate(f, g)
            continue
        want = dec_bipoly(r["result"])
        shares_factor = f and g and any(ey > 0 for (_, ey) in want)
        # coprime primitive parts: the probe; a shared factor: Brown's modular gcd + certificate
        assert P.gcd_bivariate(f, g) == want, r
        n_shared += bool(shares_factor)
        n_coprime += not shares_factor
    assert n_coprime >= 60 and n_shared >= 5


def _rand_bipoly(rng, dx, dy, c):
    return {(i, j): v for i in range(dx + 1) for j in range(dy + 1) if (v := rng.randint(-c, c))}


def test_gcd_bivariate_shared_factor_random():
    """Brown's modular gcd on f = h a, g = h b (h with a non-constant leading y-coefficient,
    contents in x and integers, lc_y vanishing at small integers) against the oracle's PRS."""
    import random
    rng = random.Random(2024)
    for t in range(24):
        h = _rand_bipoly(rng, rng.randint(0, 3), rng.randint(1, 3), 30)
        a = _rand_bipoly(rng, rng.randint(0, 3), rng.randint(0, 3), 30)
        b = _rand_bipoly(rng, rng.randint(0, 3), rng.randint(0, 3), 30)
        if t % 4 == 1:  # x-content on both sides (gcd_univariate(cf, cg) factor)
            a = O.b_mul(a, {(1, 0): 1, (0, 0): -2})
            b = O.b_mul(b, {(1, 0): 3, (0, 0): -6})
        if t % 4 == 2:  # integer contents
            a = {k: 6 * v for k, v in a.items()}
            b = {k: 10 * v for k, v in b.items()}
        if t % 4 == 3:  # lc_y(h) = x - 3: vanishes at an integer point
            dy = max(j for _, j in h)
            h = {k: v for k, v in h.items() if k[1] != dy}
            h[(1, dy)], h[(0, dy)] = 1, -3
        f, g = O.b_mul(h, a), O.b_mul(h, b)
        if not f or not g:
            continue
        assert P.gcd_bivariate(f, g) == O.gcd_bivariate(f, g), t


def test_gcd_bivariate_of_config_curve_derivatives():
    """(f_x, f_y) and (f, f_y) of BASELINE-config curves: coprime, the GPU path certifies it."""
    for kind, a, b, s in [("dense", 20, 64, 1), ("dense", 30, 128, 2), ("sheared", 3, 0, 1), ("dense", 16, 1024, 1)]:
        f = curves.make(kind, a, b, s)
        fx, fy = curves.derive_x(f), curves.derive_y(f)
        want_x = O.content_y(fx), O.content_y(fy)  # cheap: chains stop at 1
        expect = {(i, 0): c for i, c in enumerate(O.gcd_univariate(*want_x)) if c}
        assert P.gcd_bivariate(fx, fy) == expect
        assert P.gcd_bivariate(f, fy) == {(i, 0): c for i, c in
                                          enumerate(O.gcd_univariate(O.content_y(f), want_x[1])) if c}


def _teissier_curve(r):
    return curves.make(*r["curve"]) if "curve" in r else dec_bipoly(r["f"])


def test_teissier_q_against_reference():
    rows = load("teissier.jsonl")
    assert len(rows) >= 12
    for r in rows:
        f = _teissier_curve(r)
        fx, fy = curves.derive_x(f), curves.derive_y(f)
        h_ref = dec_bipoly(r["h"])
        h = P.gcd_bivariate(fx, fy)
        assert h == h_ref
        if max((ex for ex, _ in h), default=0) > 0 or max((ey for _, ey in h), default=0) > 0:
            fx, fy = O.divexact_bivariate(fx, h), O.divexact_bivariate(fy, h)
        q = P.resultant(fx, fy)
        assert q == dec_upoly(r["result"]), r.get("curve", r.get("name"))
        assert _sqf(P.yun_squarefree(q)) == dec_sqf(r["qsf"])


def test_equal_degree_fast_kernel_matches_general():
    """deg_y p == deg_y q (the Q shape) runs the EQ fast kernel; compare with the oracle
    restatement on random inputs where formal leading coefficients vanish at some points."""
    import random
    rng = random.Random(76)
    for t in range(12):
        n = rng.randint(2, 9)
        p = {(i, j): rng.randint(-99, 99) for i in range(rng.randint(1, 5)) for j in range(n + 1)}
        q = {(i, j): rng.randint(-99, 99) for i in range(rng.randint(1, 5)) for j in range(n + 1)}
        p[(0, n)] = p.get((0, n)) or 3
        q[(0, n)] = q.get((0, n)) or -5
        if t % 3 == 0:  # lc_y a polynomial in x: vanishes mod p at some evaluation points
            p[(2, n)] = 7
        p = {k: v for k, v in p.items() if v}
        q = {k: v for k, v in q.items() if v}
        assert P.resultant(p, q) == O.resultant(p, q, "y")


def test_teissier_q_big_digests():
    """Q = res(f_x, f_y) at d20/64 (EQ fast kernel, n = 19) and the sheared K=3 curve
    against sha256 digests of the reference's outputs (tests/golden/teissier_big.jsonl)."""
    import hashlib
    rows = load("teissier_big.jsonl")
    assert len(rows) == 2
    for r in rows:
        f = curves.make(*r["curve"])
        fx, fy = curves.derive_x(f), curves.derive_y(f)
        assert P.gcd_bivariate(fx, fy) == {(0, 0): 1}
        q = P.resultant(fx, fy)
        hexes = [format(c, "x") for c in q]
        assert len(q) - 1 == r["deg"] and hexes[-1] == r["lc"] and hexes[0] == r["c0"]
        assert hashlib.sha256(",".join(hexes).encode()).hexdigest() == r["sha256"], r["curve"]
