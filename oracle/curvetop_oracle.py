"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference hot path.

This module restates, in exact Python integer arithmetic, the reference
algorithms for the path this repo accelerates:

  * ``resultant``        -- /root/reference/proj/src/elim.cpp:95-136 (subresultant PRS over Z[x])
  * ``yun_squarefree``   -- elim.cpp:138-165
  * ``gcd_univariate``   -- elim.cpp:80-93 (primitive PRS)
  * ``square_free_part`` -- elim.cpp:204-210
  * ``reconstruct``      -- elim.cpp:74-78
  * ``gcd_bivariate``    -- elim.cpp:178-202 (PRS in y over Z[x] after content_y, bipoly.cpp:192-201)
  * ``curve_q``          -- CurveContext::resultant_q / q_factorization, lift.cpp:76-101
                            (h = gcd_bivariate(f_x, f_y), Q = res(f_x/h, f_y/h), Yun(Q))
  * the Z[x] substrate they use -- upoly.cpp:30-120, bipoly.cpp:103-190

Parity status: PINNED.  ``tests/test_oracle.py`` checks every function here
against the golden vectors in ``tests/golden/`` which were produced by the
reference itself (compiled unmodified into ``oracle/_ref/`` by
``oracle/Makefile``; generator script ``oracle/make_golden.py``), including
the exact random inputs of the reference's own ``proj/tests/test_elim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg may import this module, and only as the checker.  The
product (``paper_1103_4697_b200``) never imports it.

Representations: a univariate polynomial is a list of ints, low -> high, with
trailing zeros trimmed (the zero polynomial is ``[]``, degree -1; upoly.hpp:12-13,
83-85).  A bivariate polynomial is a dict ``{(deg_x, deg_y): int}`` without
zero entries (bipoly.cpp:7-15).
"""

from __future__ import annotations

from math import gcd as _igcd


class Error(RuntimeError):
    """curvetop::Error (numeric.hpp:15-18)."""


class PreconditionError(Error):
    """curvetop::PreconditionError (numeric.hpp:20-24)."""


# ----------------------------------------------------------------------------
# Univariate Z[x]  (upoly.cpp)
# ----------------------------------------------------------------------------

def trim(c):
    """upoly.hpp:83-85: drop trailing zeros."""
    c = list(c)
    while c and c[-1] == 0:
        c.pop()
    return c


def degree(p):
    return len(p) - 1


def u_add(a, b):
    n = max(len(a), len(b))
    return trim([(a[i] if i < len(a) else 0) + (b[i] if i < len(b) else 0) for i in range(n)])


def u_sub(a, b):
    n = max(len(a), len(b))
    return trim([(a[i] if i < len(a) else 0) - (b[i] if i < len(b) else 0) for i in range(n)])


def u_neg(a):
    return [-c for c in a]


def u_mul(a, b):
    """upoly.cpp:30-36 (schoolbook)."""
    if not a or not b:
        return []
    r = [0] * (len(a) + len(b) - 1)
    for i, ai in enumerate(a):
        if ai == 0:
            continue
        for j, bj in enumerate(b):
            r[i + j] += ai * bj
    return trim(r)


def u_scale(a, s):
    """upoly.cpp:38-43."""
    if s == 0:
        return []
    return [c * s for c in a]


def u_pow(p, k):
    """elim.cpp:9-13."""
    r = [1]
    for _ in range(k):
        r = u_mul(r, p)
    return r


def derivative(p):
    """upoly.cpp:45-50."""
    if len(p) <= 1:
        return []
    return trim([p[i] * i for i in range(1, len(p))])


def content(p):
    """upoly.cpp:59-66: positive gcd of all coefficients (0 for the zero poly)."""
    g = 0
    for c in p:
        g = _igcd(g, c)
        if g == 1:
            break
    return g


def _tdiv(a, b):
    """mpz_tdiv_qr semantics: quotient truncated toward zero."""
    q = abs(a) // abs(b)
    if (a < 0) != (b < 0):
        q = -q
    return q, a - q * b


def divexact_scalar(p, s):
    """upoly.cpp:75-85."""
    if s == 0:
        raise Error("divexact_scalar: zero divisor")
    out = []
    for c in p:
        q, r = _tdiv(c, s)
        if r != 0:
            raise Error("divexact_scalar: inexact division")
        out.append(q)
    return trim(out)


def primitive_positive(p):
    """upoly.cpp:68-73."""
    if not p:
        return p
    g = content(p)
    if p[-1] < 0:
        g = -g
    return divexact_scalar(p, g)


def divexact(p, d):
    """upoly.cpp:87-105 (exact polynomial division over Z)."""
    if not d:
        raise Error("divexact: zero divisor")
    if not p:
        return []
    if degree(p) < degree(d):
        raise Error("divexact: inexact division (degree)")
    rem = list(p)
    dd = degree(d)
    quo = [0] * (len(p) - len(d) + 1)
    lead = d[-1]
    for i in range(len(rem) - 1, dd - 1, -1):
        if rem[i] == 0:
            continue
        q, r = _tdiv(rem[i], lead)
        if r != 0:
            raise Error("divexact: inexact division")
        quo[i - dd] = q
        for j in range(dd + 1):
            rem[i - dd + j] -= q * d[j]
    if any(c != 0 for c in rem):
        raise Error("divexact: nonzero remainder")
    return trim(quo)


def pseudo_rem(p, d):
    """upoly.cpp:107-120: lc(d)^(deg p - deg d + 1) * p mod d."""
    if not d:
        raise Error("pseudo_rem: zero divisor")
    if not p or degree(p) < degree(d):
        return list(p)
    rem = list(p)
    lead = d[-1]
    dd = degree(d)
    for i in range(len(rem) - 1, dd - 1, -1):
        for j in range(i):
            rem[j] *= lead
        top = rem[i]
        rem[i] = 0
        for j in range(dd):
            rem[i - dd + j] -= top * d[j]
    return trim(rem[:dd])


# ----------------------------------------------------------------------------
# Bivariate Z[x,y]  (bipoly.cpp)
# ----------------------------------------------------------------------------

def b_clean(terms):
    """bipoly.cpp:7-15: drop zero coefficients."""
    return {k: v for k, v in terms.items() if v != 0}


def degree_y(f):
    return max((k[1] for k in f), default=-1)


def degree_x(f):
    return max((k[0] for k in f), default=-1)


def y_coeffs(f):
    """bipoly.cpp:109-122: dense list f_0(x), ..., f_{deg_y}(x)."""
    dy = degree_y(f)
    rows = [[] for _ in range(dy + 1)]
    for (ex, ey), c in f.items():
        r = rows[ey]
        if len(r) <= ex:
            r.extend([0] * (ex + 1 - len(r)))
        r[ex] += c
    return [trim(r) for r in rows]


def swap_vars(f):
    """bipoly.cpp:103-107."""
    return {(ey, ex): c for (ex, ey), c in f.items()}


def derive_y(f):
    """bipoly.cpp:175-190 with var = Y, order 1."""
    return b_clean({(ex, ey - 1): c * ey for (ex, ey), c in f.items() if ey >= 1})


def derive_x(f):
    return b_clean({(ex - 1, ey): c * ex for (ex, ey), c in f.items() if ex >= 1})


# ----------------------------------------------------------------------------
# Elimination  (elim.cpp)
# ----------------------------------------------------------------------------

def _yv_degree(a):
    """elim.cpp:19-23."""
    for i in range(len(a) - 1, -1, -1):
        if a[i]:
            return i
    return -1


def _yv_trim(a):
    while a and not a[-1]:
        a.pop()
    return a


def gcd_univariate(p, q):
    """elim.cpp:80-93: primitive PRS; primitive gcd with positive lc."""
    p, q = trim(p), trim(q)
    if not p and not q:
        raise PreconditionError("gcd_univariate: both inputs zero")
    if not p:
        return primitive_positive(q)
    if not q:
        return primitive_positive(p)
    a = primitive_positive(p)
    b = primitive_positive(q)
    if degree(a) < degree(b):
        a, b = b, a
    while b:
        r = primitive_positive(pseudo_rem(a, b))
        a, b = b, r
    return a


def _yv_content(a):
    """elim.cpp:29-44."""
    g = []
    for c in a:
        if not c:
            continue
        g = c if not g else gcd_univariate(g, c)
    if not g:
        return g
    ic = 0
    for c in a:
        if not c:
            continue
        ic = _igcd(ic, content(c))
    return u_scale(primitive_positive(g), ic)


def _yv_divexact_scalar(a, s):
    """elim.cpp:46-50."""
    return [c if not c else divexact(c, s) for c in a]


def _yv_prem(a, d):
    """elim.cpp:53-70: pseudo remainder in y with Z[x] coefficients."""
    da, dd = _yv_degree(a), _yv_degree(d)
    if dd < 0:
        raise Error("yv_prem: zero divisor")
    if da < dd:
        return list(a)
    rem = list(a) + [[]] * max(0, da + 1 - len(a))
    rem = rem[: da + 1]
    lead = d[dd]
    for i in range(da, dd - 1, -1):
        for j in range(i):
            rem[j] = u_mul(rem[j], lead)
        top = rem[i]
        rem[i] = []
        if top:
            for j in range(dd):
                rem[i - dd + j] = u_sub(rem[i - dd + j], u_mul(top, d[j]))
    rem = rem[:dd]
    return _yv_trim(rem)


def resultant(p, q, eliminated="y"):
    """elim.cpp:95-136: res(p, q) eliminating ``eliminated`` ('x' or 'y')."""
    if eliminated in ("x", "X"):
        return resultant(swap_vars(p), swap_vars(q), "y")
    p, q = b_clean(p), b_clean(q)
    if not p and not q:
        raise PreconditionError("resultant: both inputs identically zero")
    if not p or not q:
        return []
    n, m = degree_y(p), degree_y(q)
    if n == 0 and m == 0:
        return [1]
    if m == 0:
        return u_pow(y_coeffs(q)[0], n)
    if n == 0:
        return u_pow(y_coeffs(p)[0], m)
    a, b = y_coeffs(p), y_coeffs(q)
    sign = 1
    if n < m:
        a, b = b, a
        if (n & 1) and (m & 1):
            sign = -1
    ca, cb = _yv_content(a), _yv_content(b)
    a = _yv_divexact_scalar(a, ca)
    b = _yv_divexact_scalar(b, cb)
    scale = u_mul(u_pow(ca, _yv_degree(b)), u_pow(cb, _yv_degree(a)))
    g = [1]
    h = [1]
    while True:
        da, db = _yv_degree(a), _yv_degree(b)
        delta = da - db
        if (da & 1) and (db & 1):
            sign = -sign
        r = _yv_prem(a, b)
        if _yv_degree(r) < 0 and db > 0:
            return []
        a = b
        b = _yv_divexact_scalar(r, u_mul(g, u_pow(h, delta)))
        g = a[_yv_degree(a)]
        if delta > 0:
            h = divexact(u_pow(g, delta), u_pow(h, delta - 1))
        if _yv_degree(b) <= 0:
            break
    d = _yv_degree(a)
    res = divexact(u_pow(b[0], d), u_pow(h, d - 1))
    res = u_mul(scale, res)
    if sign < 0:
        res = u_neg(res)
    return res


def yun_squarefree(p):
    """elim.cpp:138-165.  Returns (unit, [(poly, multiplicity), ...])."""
    p = trim(p)
    if not p:
        raise PreconditionError("yun_squarefree: zero polynomial")
    P = primitive_positive(p)
    unit = content(p)
    if p[-1] < 0:
        unit = -unit
    factors = []
    if degree(P) == 0:
        return unit, factors
    dP = derivative(P)
    g = gcd_univariate(P, dP)
    if degree(g) == 0:
        return unit, [(P, 1)]
    v = divexact(P, g)
    w = divexact(dP, g)
    k = 1
    while degree(v) > 0:
        z = u_sub(w, derivative(v))
        hk = v if not z else gcd_univariate(v, z)
        if degree(hk) > 0:
            factors.append((hk, k))
        v = divexact(v, hk)
        w = z if not z else divexact(z, hk)
        k += 1
    return unit, factors


def square_free_part(p):
    """elim.cpp:204-210."""
    p = trim(p)
    if not p:
        raise PreconditionError("square_free_part: zero polynomial")
    P = primitive_positive(p)
    if degree(P) == 0:
        return P
    g = gcd_univariate(P, derivative(P))
    return P if degree(g) == 0 else primitive_positive(divexact(P, g))


def reconstruct(unit, factors):
    """elim.cpp:74-78."""
    r = [unit] if unit else []
    for poly, mult in factors:
        r = u_mul(r, u_pow(poly, mult))
    return r


# ----------------------------------------------------------------------------
# Bivariate gcd and the Teissier resultant
# ----------------------------------------------------------------------------

def from_y_coeffs(rows):
    """bipoly.cpp from_y_coeffs: {(x, y): c}."""
    return b_clean({(ex, ey): c for ey, r in enumerate(rows) for ex, c in enumerate(r)})


def content_y(f):
    """bipoly.cpp:192-201: gcd_univariate chain over the y-coefficients (stops at 1), then
    primitive_positive(g) * content(g) -- the chain's gcd with positive leading coefficient."""
    if not f:
        raise PreconditionError("content_y: zero polynomial")
    g = []
    for fi in y_coeffs(f):
        if not fi:
            continue
        g = fi if not g else gcd_univariate(g, fi)
        if g == [1]:
            break
    return u_scale(primitive_positive(g), content(g))


def divexact_univariate_x(f, d):
    """bipoly.cpp:236-244."""
    return from_y_coeffs([r if not r else divexact(r, d) for r in y_coeffs(f)])


def gcd_bivariate(f, g):
    """elim.cpp:178-202."""
    f, g = b_clean(f), b_clean(g)
    if not f and not g:
        raise PreconditionError("gcd_bivariate: both inputs zero")
    if not f:
        return g
    if not g:
        return f
    cf, cg = content_y(f), content_y(g)
    a = y_coeffs(divexact_univariate_x(f, cf))
    b = y_coeffs(divexact_univariate_x(g, cg))
    if _yv_degree(a) < _yv_degree(b):
        a, b = b, a
    while _yv_degree(b) >= 0:
        r = _yv_prem(a, b)
        c = _yv_content(r)
        a = b
        b = [] if not c else _yv_divexact_scalar(r, c)
    ca = _yv_content(a)
    pp = _yv_divexact_scalar(a, ca)
    res = b_mul(from_y_coeffs(pp), {(i, 0): c for i, c in enumerate(gcd_univariate(cf, cg)) if c})
    lead = y_coeffs(res)[degree_y(res)]
    if lead[-1] < 0:
        res = {k: -v for k, v in res.items()}
    return res


def b_mul(f, g):
    out = {}
    for (a, b), c in f.items():
        for (d, e), v in g.items():
            out[(a + d, b + e)] = out.get((a + d, b + e), 0) + c * v
    return b_clean(out)


def divexact_bivariate(p, d):
    """bipoly.cpp:246-266: long division in y over Z[x], every quotient exact."""
    if not d:
        raise Error("divexact: zero divisor")
    if not p:
        return p
    if degree_y(d) == 0:
        return divexact_univariate_x(p, y_coeffs(d)[0])
    rem = y_coeffs(p)
    dc = y_coeffs(d)
    dn, dl = len(dc) - 1, dc[-1]
    if len(rem) - 1 < dn:
        raise Error("divexact: inexact division (degree)")
    quo = [[] for _ in range(len(rem) - dn)]
    for i in range(len(rem) - 1, dn - 1, -1):
        if not rem[i]:
            continue
        q = divexact(rem[i], dl)
        quo[i - dn] = q
        for j in range(dn + 1):
            rem[i - dn + j] = u_sub(rem[i - dn + j], u_mul(q, dc[j]))
    if any(r for r in rem):
        raise Error("divexact: inexact division")
    return from_y_coeffs(quo)


def curve_q(f):
    """lift.cpp:76-101: (h, Q, Yun(Q)) with h = gcd_bivariate(f_x, f_y), Q = res(f_x*, f_y*)."""
    fx, fy = derive_x(f), derive_y(f)
    if not fx:
        q = [1]
        h = {}
    else:
        h = gcd_bivariate(fx, fy)
        if degree_x(h) > 0 or degree_y(h) > 0:
            fx, fy = divexact_bivariate(fx, h), divexact_bivariate(fy, h)
        q = resultant(fx, fy, "y")
    return h, q, yun_squarefree(q)
