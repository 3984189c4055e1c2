"""GPU parity of res(p, q) through the C ABI against the reference's own outputs.

Expected values come from the reference compiled unmodified (tests/golden/, made by
oracle/make_golden.py).  Bit-exact equality of every coefficient is required.
"""

import hashlib

import pytest

import paper_1103_4697_b200 as P
from golden_io import dec_bipoly, dec_upoly, load
from paper_1103_4697_b200 import curves

pytestmark = pytest.mark.gpu


def _res(row):
    args = [dec_bipoly(a) for a in row["args"]]
    if row["op"] == "resultant_fy":
        return P.resultant(args[0], curves.derive_y(args[0]))
    return P.resultant(args[0], args[1], "x" if row["op"] == "resultant_x" else "y")


@pytest.mark.parametrize("name", ["worked.jsonl", "resultant_random.jsonl"])
def test_fixture_resultants(name):
    rows = [r for r in load(name) if r["op"].startswith("resultant")]
    assert rows
    for r in rows:
        if "error" in r:
            with pytest.raises(P.PreconditionError):
                _res(r)
        else:
            assert _res(r) == dec_upoly(r["result"]), r


def test_reference_test_elim_random_pairs():
    rows = [r for r in load("elim_cases.jsonl") if r["case"].startswith(("sylvester", "common", "generic"))]
    assert len(rows) == 200
    for r in rows:
        assert P.resultant(dec_bipoly(r["p"]), dec_bipoly(r["q"])) == dec_upoly(r["result"])


def test_small_configs():
    rows = load("configs_small.jsonl")
    assert rows
    for r in rows:
        kind, a, b, s = r["curve"]
        f = curves.make(kind, a, b, s)
        assert P.resultant(f, curves.derive_y(f)) == dec_upoly(r["result"]), r["curve"]


def _digest(coeffs):
    return hashlib.sha256(",".join(format(c, "x") for c in coeffs).encode()).hexdigest()


@pytest.mark.parametrize("row", load("configs_big.jsonl"), ids=lambda r: "_".join(map(str, r["curve"])))
def test_big_configs_digest(row):
    kind, a, b, s = row["curve"]
    f = curves.make(kind, a, b, s)
    R = P.resultant(f, curves.derive_y(f))
    assert len(R) - 1 == row["deg"]
    assert format(R[-1], "x") == row["lc"] and format(R[0], "x") == row["c0"]
    assert _digest(R) == row["sha256"]


def test_batch_api_mixed_shapes():
    """ctg_resultant_batch groups same-shape problems into one batched plan; mixed shapes,
    zero operands and Var::X must still match the reference one by one."""
    rows = [r for r in load("resultant_random.jsonl") if r["op"] == "resultant_y" and "error" not in r]
    rows += [r for r in load("worked.jsonl") if r["op"] == "resultant_y" and "error" not in r]
    pairs = [(dec_bipoly(r["args"][0]), dec_bipoly(r["args"][1])) for r in rows]
    got = P.resultant_batch(pairs)
    assert got == [dec_upoly(r["result"]) for r in rows]


def test_batch_plan_same_shape_curves():
    small = [r for r in load("configs_small.jsonl") if r["curve"][:3] == ["dense", 10, 10]]
    assert len(small) == 5
    pairs = []
    for r in small:
        f = curves.make(*r["curve"])
        pairs.append((f, curves.derive_y(f)))
    got = P.resultant_batch(pairs)
    assert got == [dec_upoly(r["result"]) for r in small]


def _term_orders(f, rng):
    """The same polynomial as raw CSR operands in several term orders and encodings."""
    items = [(k[0], k[1], v) for k, v in f.items() if v]
    yx = sorted(items, key=lambda t: (t[1], t[0]))
    shuffled = items[:]
    rng.shuffle(shuffled)
    # every coefficient split into two duplicate-key terms, plus explicit zero terms
    split = []
    for dx, dy, v in shuffled:
        a = rng.randrange(-abs(v) - 5, abs(v) + 5)
        split += [(dx, dy, a), (dx, dy, v - a), (dx + 1, dy, 0)]
    # a term cancelled by a duplicate: (dx, dy) present with total zero
    split += [(0, 0, 7), (0, 0, -7)] if (0, 0) not in f else []
    return {"xy": P.HostBipoly.from_terms(sorted(items)), "yx": P.HostBipoly.from_terms(yx),
            "yx_padded": P.HostBipoly.from_terms(yx, pad_limbs=2),
            "shuffled": P.HostBipoly.from_terms(shuffled), "split_dups_zeros": P.HostBipoly.from_terms(split)}


def test_input_term_order_and_duplicates():
    """ctg_bipoly with unsorted, duplicated, zero and zero-padded terms: the parse sums
    equal keys and drops zeros (bipoly.cpp map insertion) -- same result as the canonical form."""
    import random
    rng = random.Random(5)
    rows = [r for r in load("resultant_random.jsonl") if r["op"] == "resultant_y" and "error" not in r][:12]
    rows += [r for r in load("resultant_random.jsonl") if r["op"] == "resultant_x" and "error" not in r][:6]
    assert rows
    for r in rows:
        f, g = (dec_bipoly(a) for a in r["args"])
        var = "x" if r["op"] == "resultant_x" else "y"
        want = dec_upoly(r["result"])
        fo, go = _term_orders(f, rng), _term_orders(g, rng)
        for kind in fo:
            assert P.resultant_host(fo[kind], go[kind], var) == want, (kind, r)
    # the f_y shape (derivative detection) through the permuted encodings
    f = curves.make("dense", 8, 40, 3)
    want = P.resultant(f, curves.derive_y(f))
    fo, go = _term_orders(f, rng), _term_orders(curves.derive_y(f), rng)
    for kind in fo:
        assert P.resultant_host(fo[kind], go[kind]) == want, kind


def _eval_x(f, x0):
    """f(x0, y) as a bivariate of x-degree 0."""
    out = {}
    for (ex, ey), c in f.items():
        out[(0, ey)] = out.get((0, ey), 0) + c * x0 ** ex
    return {k: v for k, v in out.items() if v}


@pytest.mark.parametrize("d", [44, 60])
def test_specialisation_beyond_fast_degrees(d):
    """deg_y > 40 runs the general formal-degree kernel for every unit.  R(x0) must equal
    res_y(f(x0, y), f_y(x0, y)) (lc_y f constant: specialisation commutes),
    checked exactly with the oracle restatement on the univariate specialisations."""
    import curvetop_oracle as O
    f = curves.make("dense", d, 8, 7)
    R = P.resultant(f, curves.derive_y(f))
    assert len(R) - 1 <= d * (d - 1)
    for x0 in (0, 1, -2, 3):
        fx0 = _eval_x(f, x0)
        want = O.resultant(fx0, O.derive_y(fx0), "y")
        got = sum(c * x0 ** i for i, c in enumerate(R))
        assert [got] == want or (got == 0 and want == []), x0


_FUSED_CHILD = r"""
import hashlib, json, sys
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/tests"]
import paper_1103_4697_b200 as P
from golden_io import dec_bipoly, dec_upoly, load
from paper_1103_4697_b200 import curves
n = 0
for r in load("configs_small.jsonl"):
    f = curves.make(*r["curve"])
    assert P.resultant(f, curves.derive_y(f)) == dec_upoly(r["result"]), r["curve"]
    n += 1
for r in load("resultant_random.jsonl"):
    if r["op"] == "resultant_fy" and "error" not in r:
        f = dec_bipoly(r["args"][0])
        assert P.resultant(f, curves.derive_y(f)) == dec_upoly(r["result"]), r
        n += 1
for r in load("configs_big.jsonl"):
    if True:
        f = curves.make(*r["curve"])
        R = P.resultant(f, curves.derive_y(f))
        h = hashlib.sha256(",".join(format(c, "x") for c in R).encode()).hexdigest()
        assert h == r["sha256"], r["curve"]
        n += 1
print(json.dumps({"checked": n, "launches": P.last_call_stats()["kernel_launches"]}))
"""


def test_fused_k2_k3_kernel():
    """The opt-in fused evaluation + Euclid kernel (CTG_FUSE=1, read once per process) on the
    res(f, f_y) fixtures and the reference digests of the four big configs."""
    import json
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CTG_FUSE="1")
    out = subprocess.run([sys.executable, "-c", _FUSED_CHILD, repo], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["checked"] >= 6


def test_batch_streaming_blocks_mixed():
    """The streaming batch path (small head / tail blocks, large middle blocks, two compute
    streams, regions sized from the first plan): a long batch interleaving same-shape curves,
    other shapes, zero operands and a first block smaller than the later plans, against the
    reference's fixtures and one-shot calls."""
    import random
    rng = random.Random(5)
    fixtures = [r for r in load("resultant_random.jsonl") if r["op"] == "resultant_y" and "error" not in r]
    items, want = [], []
    # a head of small curves (the first plan sizes the regions), then bigger ones (regrow)
    for s in range(1, 40):
        f = curves.make("dense", 6, 10, s)
        items.append((f, curves.derive_y(f)))
        want.append(None)
    for t in range(160):
        c = rng.random()
        if c < 0.35:
            r = rng.choice(fixtures)
            items.append((dec_bipoly(r["args"][0]), dec_bipoly(r["args"][1])))
            want.append(dec_upoly(r["result"]))
        elif c < 0.4:
            items.append(({}, {(0, 1): 3}))  # one zero operand -> zero polynomial
            want.append([])
        else:
            f = curves.make("dense", rng.choice([8, 12, 16]), rng.choice([10, 64]), rng.randint(1, 9))
            items.append((f, curves.derive_y(f)))
            want.append(None)
    got = P.resultant_batch(items)
    assert len(got) == len(items)
    for (p, q), g, w in zip(items, got, want):
        assert g == (w if w is not None else P.resultant(p, q))
    # sizes around the block boundaries
    for n in (1, 31, 32, 33, 64, 65):
        sub = items[:n]
        assert P.resultant_batch(sub) == got[:n]


def test_batch_error_in_a_late_block():
    """Both operands zero in a late block: PreconditionError for the whole call (earlier
    blocks already ran on the GPU; their results are released), and the library stays usable."""
    items = []
    for s in range(1, 80):
        f = curves.make("dense", 6, 10, s)
        items.append((f, curves.derive_y(f)))
    items.append(({}, {}))
    with pytest.raises(P.PreconditionError):
        P.resultant_batch(items)
    assert P.resultant_batch(items[:3]) == [P.resultant(*it) for it in items[:3]]


def test_concurrent_calls_from_threads():
    """Entry points are re-entrant (SURVEY §8(b) threading row): resultants, batches, Yun and
    gcds issued from several host threads at once (ctypes drops the GIL during the calls) give
    the single-threaded results."""
    import threading
    fs = [curves.make("dense", d, 16, s) for d, s in [(8, 1), (10, 2), (12, 3), (9, 4)]]
    pairs = [(f, curves.derive_y(f)) for f in fs]
    want_r = [P.resultant(*pq) for pq in pairs]
    want_y = [P.yun_squarefree(r) for r in want_r]
    want_g = P.gcd_univariate(want_r[0], want_r[1])
    errors = []

    def work(t):
        try:
            for it in range(6):
                i = (t + it) % len(pairs)
                assert P.resultant(*pairs[i]) == want_r[i]
                assert P.yun_squarefree(want_r[i]) == want_y[i]
                assert P.resultant_batch(pairs) == want_r
                assert P.gcd_univariate(want_r[0], want_r[1]) == want_g
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ths = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errors, errors[0]


def test_crt_beyond_tensor_core_prime_count():
    """More than kI8MaxPrimes = 8192 primes (the u8 GEMM's s32 exactness limit): dense degree 3
    with 65,536-bit coefficients needs ~10,900 primes and takes the IMAD CRT path; exact
    against the oracle restatement of the reference's PRS."""
    import curvetop_oracle as O
    f = curves.make("dense", 3, 65536, 3)
    R = P.resultant(f, curves.derive_y(f))
    assert P.last_call_stats()["n_primes"] > 8192
    assert R == O.resultant(f, O.derive_y(f), "y")


def test_large_batch_bounded_slots():
    """600 curves: many more chunks than pipeline slots (each slot reused every third chunk,
    memory bounded by the largest block), results identical to one-at-a-time calls."""
    pairs = []
    for s in range(1, 601):
        f = curves.make("dense", 6 + s % 3, 12, s)
        pairs.append((f, curves.derive_y(f)))
    got = P.resultant_batch(pairs)
    for i in range(0, 600, 37):
        assert got[i] == P.resultant(*pairs[i]), i
    assert got[:64] == P.resultant_batch(pairs[:64])


_HYB_EXTRA = r"""
import hashlib, json, sys
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/tests"]
import paper_1103_4697_b200 as P
from paper_1103_4697_b200 import curves
out = {}
for d in (4, 9, 16, 20, 25, 32):
    f = curves.make("dense", d, 40, d)
    R = P.resultant(curves.derive_x(f), curves.derive_y(f))  # equal y-degrees: the EQ kernel
    out[str(d)] = hashlib.sha256(",".join(format(c, "x") for c in R).encode()).hexdigest()
print(json.dumps(out))
"""


def test_k3_hybrid_euclid():
    """The opt-in hybrid FP64-quotient / IMAD Euclid (CTG_K3_HYB=1, read once per process):
    every res(f, f_y) fixture, the reference digests of the big configs, and the equal-degree
    (Teissier-shape) kernel against the default Montgomery path."""
    import json
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CTG_K3_HYB="1")
    out = subprocess.run([sys.executable, "-c", _FUSED_CHILD, repo], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert json.loads(out.stdout.strip().splitlines()[-1])["checked"] >= 6
    out = subprocess.run([sys.executable, "-c", _HYB_EXTRA, repo], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    got = json.loads(out.stdout.strip().splitlines()[-1])
    for d, h in got.items():
        f = curves.make("dense", int(d), 40, int(d))
        assert _digest(P.resultant(curves.derive_x(f), curves.derive_y(f))) == h, d


def _upow_mul(g, e, c):
    """c * g(x)^e over Z (dense low -> high)."""
    out = [c]
    for _ in range(e):
        nxt = [0] * (len(out) + len(g) - 1)
        for i, a in enumerate(out):
            for j, b in enumerate(g):
                nxt[i + j] += a * b
        out = nxt
    return out


def test_flag_list_overflow_superelliptic():
    """y^n + g(x): the remainder sequence drops degree at EVERY (prime, point) unit, so the fast
    kernel flags all of them (515 primes x 256 points > the 65,536-entry flag list).
    res(y^n + g, n y^(n-1)) = n^n g^(n-1) exactly (the reference's Sylvester convention,
    test_elim.cpp:16: res(y^2 - x, 2y) = -4x)."""
    import random
    rng = random.Random(1103)
    g = [rng.getrandbits(1024) * rng.choice((-1, 1)) for _ in range(17)]
    f = {(i, 0): c for i, c in enumerate(g) if c}
    f[(0, 16)] = 1
    assert P.resultant(f, curves.derive_y(f)) == _upow_mul(g, 15, 16 ** 16)


def test_flag_list_overflow_batch():
    """64 curves y^20 + g_b(x) in one batched plan: ~295K flagged units in one launch."""
    import random
    rng = random.Random(4697)
    pairs, want = [], []
    for _ in range(64):
        g = [rng.randint(-1023, 1023) or 1 for _ in range(21)]
        f = {(i, 0): c for i, c in enumerate(g)}
        f[(0, 20)] = 1
        pairs.append((f, curves.derive_y(f)))
        want.append(_upow_mul(g, 19, 20 ** 20))
    assert P.resultant_batch(pairs) == want


def test_spec_sylvester_acceptance_500_pairs():
    """SPEC.md:632 acceptance #2 on the GPU path: resultant == Sylvester determinant on 500 random
    pairs (deg <= 6, |c| <= 2^16), zero mismatches.  The fixture holds the reference's resultant
    digests, which make_golden.py asserted equal to the reference's Bareiss oracle
    (proj/tests/oracles.cpp:82-120).  Both the batched call (shapes grouped) and single calls."""
    rows = load("sylvester_acceptance.jsonl")
    assert len(rows) >= 500
    pairs = [(dec_bipoly(r["p"]), dec_bipoly(r["q"])) for r in rows]
    got = P.resultant_batch(pairs)
    for r, R in zip(rows, got):
        assert len(R) - 1 == r["deg"] and _digest(R) == r["sha256"], r
    for r, pq in list(zip(rows, pairs))[::10]:
        assert _digest(P.resultant(*pq)) == r["sha256"]
