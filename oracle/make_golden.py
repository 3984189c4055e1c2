"""TEST INFRASTRUCTURE ONLY: generate the golden fixtures under tests/golden/.

Every expected output in tests/golden/ comes from the reference itself
(/root/reference/proj compiled unmodified into oracle/_ref/ by oracle/Makefile)
via ``oracle/_ref/refdriver``.  Run in the build container (it needs the
reference build; the GPU box only reads the committed fixtures):

    make -C oracle all
    python oracle/make_golden.py            # small fixtures (seconds)
    python oracle/make_golden.py --big      # + full-size digests (d30/128 takes ~30 min of CPU)

Fixture files (JSON lines):
  elim_cases.jsonl      exact random inputs of proj/tests/test_elim.cpp (seeds 21-24) + outputs
  worked.jsonl          the hand-written examples of test_elim.cpp / SPEC.md:121-147 + conventions
  resultant_random.jsonl  extra random resultant shapes (formal-degree drops, n<m, Var::X, big coeffs)
  univariate_random.jsonl yun / gcd / square_free_part on structured random inputs
  configs_small.jsonl   res(f, f_y) (+ Yun) on the BASELINE configs that finish in seconds
  configs_big.jsonl     sha256 digests of res(f, f_y) at the full BASELINE sizes
  bivariate_gcd.jsonl   gcd_bivariate (elim.cpp:178-202) on coprime / content-sharing / factor-sharing pairs
  sylvester_acceptance.jsonl  SPEC.md:632: resultant == Sylvester determinant (oracles.cpp:82-120), 500 pairs
  teissier.jsonl        CurveContext::resultant_q + q_factorization (lift.cpp:76-101): h = gcd(f_x, f_y),
                        Q = res(f_x / h, f_y / h), Yun(Q) -- SURVEY.md §8(f) rank 1
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import random
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

from paper_1103_4697_b200 import curves  # noqa: E402

DRIVER = os.path.join(HERE, "_ref", "refdriver")
GOLD = os.path.join(REPO, "tests", "golden")


def hx(v: int) -> str:
    return format(v, "x")


def req_bipoly(f: dict) -> str:
    lines = [f"B {len(f)}"]
    for (ex, ey), c in sorted(f.items()):
        lines.append(f"{ex} {ey} {hx(c)}")
    return "\n".join(lines)


def req_upoly(p: list) -> str:
    return "\n".join([f"U {len(p)}"] + [hx(c) for c in p])


def run_batch(requests: list[tuple[str, list]]) -> list[dict]:
    """requests: (op, [operand, ...]) with dict operands (bivariate) or list operands."""
    text = []
    for op, args in requests:
        text.append(f"OP {op}")
        for a in args:
            text.append(req_bipoly(a) if isinstance(a, dict) else req_upoly(a))
        text.append("END")
    out = subprocess.run([DRIVER, "batch"], input="\n".join(text) + "\n", capture_output=True, text=True,
                         check=True).stdout
    return [json.loads(l) for l in out.splitlines() if l.strip()]


def enc_bipoly(f: dict) -> list:
    return [[ex, ey, hx(c)] for (ex, ey), c in sorted(f.items())]


def enc_upoly(p: list) -> list:
    return [hx(c) for c in p]


def write(name: str, rows: list[dict]) -> None:
    os.makedirs(GOLD, exist_ok=True)
    with open(os.path.join(GOLD, name), "w") as fh:
        for r in rows:
            fh.write(json.dumps(r, separators=(",", ":")) + "\n")
    print(f"wrote {name}: {len(rows)} rows")


def emit(requests, meta=None) -> list[dict]:
    res = run_batch(requests)
    rows = []
    for i, ((op, args), r) in enumerate(zip(requests, res)):
        row = {"op": op, "args": [enc_bipoly(a) if isinstance(a, dict) else enc_upoly(a) for a in args]}
        if meta:
            row.update(meta[i])
        if "error" in r:
            row["error"] = r["error"]
        else:
            row["result"] = r["result"]
        row["ref_seconds"] = r["seconds"]
        rows.append(row)
    return rows


def bp(*terms) -> dict:
    out: dict = {}
    for ex, ey, c in terms:
        out[(ex, ey)] = out.get((ex, ey), 0) + c
    return {k: v for k, v in out.items() if v}


def worked() -> list[dict]:
    parab = bp((0, 2, 1), (1, 0, -1))
    two_y = bp((0, 1, 2))
    circle = bp((2, 0, 1), (0, 2, 1), (0, 0, -1))
    cusp = bp((0, 2, 1), (3, 0, -1))
    hyper = bp((1, 1, 1), (0, 0, -1))
    fy = bp((1, 0, 1))
    line = bp((1, 0, 1), (0, 1, -1))
    reqs = [
        ("resultant_y", [parab, two_y]),          # test_elim.cpp:16  -4x
        ("resultant_y", [circle, two_y]),         # :19  4x^2 - 4
        ("resultant_y", [cusp, two_y]),           # :22  -4x^3
        ("resultant_y", [hyper, fy]),             # :28  x
        ("resultant_y", [fy, fy]),                # :29  1
        ("resultant_y", [hyper, {}]),             # :30  0
        ("resultant_y", [{}, {}]),                # :31  PreconditionError
        ("resultant_x", [parab, line]),           # :76
        ("resultant_fy", [circle]),
        ("resultant_fy", [cusp]),
        ("resultant_fy", [bp((1, 1, 1), (0, 0, -1))]),  # lc_y = x vanishes at x = 0
        ("yun", [[0, 0, 1, 1]]),                  # :82
        ("yun", [[-2, 0, 1]]),                    # :90
        ("yun", [[-1, 3, -3, 1]]),                # :97
        ("yun", [[]]),                            # :102 PreconditionError
        ("yun", [[-4, 0, 4]]),                    # :147
        ("yun", [[0, 0, 0, -4]]),                 # :151
        ("yun", [[0, 0, -4, -4]]),                # :156
        ("yun", [[5]]),
        ("yun", [[-6]]),
        ("gcd", [[-2, 0, 1], [-2, 0, 1]]),        # :126
        ("gcd", [[-1, 0, 1], [-1, 1]]),           # :127
        ("gcd", [[-2, 0, 1], [-3, 0, 1]]),        # :128
        ("gcd", [[], [6, -4]]),
        ("gcd", [[], []]),
        ("gcd", [[12], [18]]),
        ("sqfp", [[0, 0, 1, 1]]),
        ("sqfp", [[-1, 3, -3, 1]]),
        ("sqfp", [[]]),
        ("sqfp", [[7]]),
    ]
    return emit(reqs)


def rand_bipoly(rng: random.Random, dx: int, dy: int, bits: int, density: float = 1.0) -> dict:
    f = {}
    for i in range(dx + 1):
        for j in range(dy + 1):
            if rng.random() > density:
                continue
            c = rng.getrandbits(bits) * rng.choice((-1, 1))
            if c:
                f[(i, j)] = c
    return f


def resultant_random() -> list[dict]:
    rng = random.Random(1103_4697)
    reqs, meta = [], []
    for t in range(160):
        kind = t % 8
        if kind == 0:     # dense-ish, moderate bits
            p = rand_bipoly(rng, rng.randint(0, 4), rng.randint(1, 5), rng.randint(1, 40))
            q = rand_bipoly(rng, rng.randint(0, 4), rng.randint(1, 5), rng.randint(1, 40))
        elif kind == 1:   # big coefficients
            p = rand_bipoly(rng, rng.randint(0, 3), rng.randint(1, 4), rng.randint(100, 400))
            q = rand_bipoly(rng, rng.randint(0, 3), rng.randint(1, 4), rng.randint(100, 400))
        elif kind == 2:   # sparse, lc_y(p) a polynomial in x (formal-degree drops at points)
            p = rand_bipoly(rng, rng.randint(1, 5), rng.randint(1, 5), 8, 0.5)
            q = rand_bipoly(rng, rng.randint(1, 5), rng.randint(1, 5), 8, 0.5)
        elif kind == 3:   # n < m (swap + sign)
            p = rand_bipoly(rng, 2, rng.randint(1, 3), 12)
            q = rand_bipoly(rng, 2, rng.randint(4, 6), 12)
        elif kind == 4:   # p, p_y with lc_y = x^k style
            p = rand_bipoly(rng, rng.randint(1, 4), rng.randint(2, 6), 16, 0.7)
            q = curves.derive_y(p)
        elif kind == 5:   # common factor -> 0
            c = rand_bipoly(rng, 1, rng.randint(1, 2), 4)
            p = curves._bmul(rand_bipoly(rng, 1, 2, 4), c)
            q = curves._bmul(rand_bipoly(rng, 1, 2, 4), c)
        elif kind == 6:   # one side of degree 0 in y
            p = rand_bipoly(rng, rng.randint(0, 3), rng.randint(1, 4), 20)
            q = rand_bipoly(rng, rng.randint(0, 3), 0, 20)
        else:             # univariate-only x content
            g = rand_bipoly(rng, 2, 0, 6)
            p = curves._bmul(rand_bipoly(rng, 2, rng.randint(1, 4), 10), g)
            q = curves._bmul(rand_bipoly(rng, 2, rng.randint(1, 4), 10), g)
        if not p and not q:
            continue
        op = "resultant_x" if (t % 11 == 3) else "resultant_y"
        reqs.append((op, [p, q]))
        meta.append({"kind": kind})
    return emit(reqs, meta)


def rand_upoly(rng: random.Random, deg: int, bits: int) -> list:
    c = [rng.getrandbits(bits) * rng.choice((-1, 1)) for _ in range(deg + 1)]
    while c and c[-1] == 0:
        c[-1] = rng.getrandbits(bits) or 1
    return c


def umul(a, b):
    if not a or not b:
        return []
    r = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            r[i + j] += x * y
    while r and r[-1] == 0:
        r.pop()
    return r


def univariate_random() -> list[dict]:
    rng = random.Random(4697)
    reqs = []
    for t in range(60):   # Yun on products with repeated factors
        parts = [rand_upoly(rng, rng.randint(1, 4), rng.randint(2, 30)) for _ in range(rng.randint(1, 4))]
        p = [rng.choice((-1, 1)) * rng.randint(1, 50)]
        for i, part in enumerate(parts):
            for _ in range(rng.randint(1, 4)):
                p = umul(p, part)
        reqs.append(("yun", [p]))
        reqs.append(("sqfp", [p]))
    for t in range(60):   # gcd with a planted common factor
        w = rand_upoly(rng, rng.randint(0, 5), rng.randint(2, 40))
        u = rand_upoly(rng, rng.randint(0, 6), rng.randint(2, 40))
        v = rand_upoly(rng, rng.randint(0, 6), rng.randint(2, 40))
        reqs.append(("gcd", [umul(u, w), umul(v, w)]))
    return emit(reqs)


def configs_small() -> list[dict]:
    reqs, meta = [], []
    for (kind, a, b, seeds, yun) in [("dense", 6, 10, (1, 2, 3), True), ("dense", 8, 10, (1,), True),
                                     ("dense", 10, 10, (1, 2, 3, 4, 5), True),
                                     ("sheared", 2, 0, (1, 2), True), ("dense", 12, 40, (1,), False),
                                     ("dense", 5, 300, (1,), True)]:
        for s in seeds:
            f = curves.make(kind, a, b, s)
            reqs.append(("resultant_fy", [f]))
            meta.append({"curve": [kind, a, b, s], "with_yun": yun})
    rows = emit(reqs, meta)
    yreq, yidx = [], []
    for i, r in enumerate(rows):
        if r.get("with_yun"):
            yreq.append(("yun", [[int(c, 16) for c in r["result"]]]))
            yidx.append(i)
    for i, y in zip(yidx, run_batch(yreq)):
        rows[i]["yun"] = y["result"]
        rows[i]["yun_ref_seconds"] = y["seconds"]
    for r in rows:
        del r["args"]  # curve is regenerated from (kind, a, b, seed)
    return rows


def digest(coeffs_hex: list) -> str:
    return hashlib.sha256(",".join(coeffs_hex).encode()).hexdigest()


def configs_big(cache_dir: str, cached_only: bool = False) -> list[dict]:
    """Digests of the reference's R at the full BASELINE sizes, seeds 1..: outputs cached by
    oracle/gen_big.py (parallel runs of oracle/_ref/refdriver), rows already in the committed
    file are kept when their cache is gone."""
    import gen_big
    old = {}
    path = os.path.join(GOLD, "configs_big.jsonl")
    if os.path.exists(path):
        for line in open(path):
            r = json.loads(line)
            old[tuple(r["curve"])] = r
    todo = [("dense", 20, 64, 1, False), ("sheared", 3, 0, 1, True), ("dense", 16, 1024, 1, False),
            ("dense", 30, 128, 1, False)] + [t[:5] for t in gen_big.PLAN]
    rows = []
    for (kind, a, b, s, with_yun) in todo:
        name = gen_big.cache_name(kind, a, b, s)
        cached = os.path.join(cache_dir, f"out_{name}.txt")
        lines = []
        if os.path.exists(cached) and os.path.getsize(cached) > 0:
            lines = open(cached).read().splitlines()
            r = json.loads(lines[0])
        elif (kind, a, b, s) in old:
            rows.append(old[(kind, a, b, s)])
            continue
        elif cached_only:
            print(f"skip {name}: no cached reference output")
            continue
        else:
            f = curves.make(kind, a, b, s)
            r = run_batch([("resultant_fy", [f])])[0]
        res = r["result"]
        ints = [int(c, 16) for c in res]
        row = {"curve": [kind, a, b, s], "deg": len(res) - 1, "max_bits": max(abs(c).bit_length() for c in ints),
               "sha256": digest(res), "lc": res[-1], "c0": res[0], "ref_seconds": r["seconds"]}
        if with_yun:
            y = json.loads(lines[1])["result"] if len(lines) > 1 else run_batch([("yun", [ints])])[0]["result"]
            row["yun_unit"] = y["unit"]
            row["yun"] = [{"mult": fct["mult"], "deg": len(fct["poly"]) - 1, "sha256": digest(fct["poly"])}
                          for fct in y["factors"]]
        rows.append(row)
    return rows


def bivariate_gcd() -> list[dict]:
    rng = random.Random(178_202)
    reqs, meta = [], []
    for t in range(90):
        kind = t % 9
        if kind == 0:     # generic coprime pair
            f = rand_bipoly(rng, rng.randint(0, 4), rng.randint(1, 5), rng.randint(2, 40))
            g = rand_bipoly(rng, rng.randint(0, 4), rng.randint(1, 5), rng.randint(2, 40))
        elif kind == 1:   # x-contents sharing a factor, coprime primitive parts
            c = rand_bipoly(rng, rng.randint(1, 3), 0, 6)
            f = curves._bmul(rand_bipoly(rng, 2, rng.randint(1, 4), 10), curves._bmul(c, rand_bipoly(rng, 1, 0, 5)))
            g = curves._bmul(rand_bipoly(rng, 2, rng.randint(1, 4), 10), c)
        elif kind == 2:   # integer contents only (gcd_univariate drops them)
            k1, k2 = rng.randint(2, 30), rng.randint(2, 30)
            f = {e: k1 * v for e, v in rand_bipoly(rng, 2, rng.randint(1, 3), 8).items()}
            g = {e: k2 * v for e, v in rand_bipoly(rng, 2, rng.randint(1, 3), 8).items()}
        elif kind == 3:   # one operand of degree 0 in y
            f = rand_bipoly(rng, rng.randint(0, 4), rng.randint(1, 4), 12)
            g = rand_bipoly(rng, rng.randint(1, 4), 0, 12)
        elif kind == 4:   # single y-coefficient operands (content = the coefficient itself)
            f = {(ex, 3): v for (ex, _), v in rand_bipoly(rng, 3, 0, 10).items()}
            g = rand_bipoly(rng, 2, 2, 10)
        elif kind == 5:   # common bivariate factor (primitive parts NOT coprime)
            c = rand_bipoly(rng, rng.randint(0, 2), rng.randint(1, 2), 5)
            f = curves._bmul(rand_bipoly(rng, 2, rng.randint(1, 3), 6), c)
            g = curves._bmul(rand_bipoly(rng, 2, rng.randint(1, 3), 6), c)
        elif kind == 6:   # (f, f_y) of random curves, lc_y depending on x
            f = rand_bipoly(rng, rng.randint(1, 5), rng.randint(2, 6), 16, 0.7)
            g = curves.derive_y(f)
        elif kind == 7:   # (f_x, f_y) of dense curves
            f0 = curves.make("dense", rng.randint(3, 7), 10, rng.randint(1, 99))
            f, g = curves.derive_x(f0), curves.derive_y(f0)
        else:             # a zero operand / negative leading coefficients
            f = {e: -v for e, v in rand_bipoly(rng, 2, 2, 10).items()}
            g = {} if t % 2 else {e: -abs(v) for e, v in rand_bipoly(rng, 1, 1, 10).items()}
        if not f and not g:
            continue
        reqs.append(("gcd_bivariate", [f, g]))
        meta.append({"kind": kind})
    rows = emit(reqs, meta)
    reqs = [("gcd_bivariate", [{}, {}])]
    rows += emit(reqs, [{"kind": "both_zero"}])
    return rows


def teissier_curves() -> list:
    out = [("dense", 6, 10, s) for s in (1, 2, 3)] + [("dense", 8, 10, 1), ("dense", 10, 10, 1),
                                                       ("sheared", 2, 0, 1), ("dense", 5, 300, 1)]
    return out


def special_curves() -> dict:
    s = lambda *t: bp(*t)
    return {
        "circle": s((2, 0, 1), (0, 2, 1), (0, 0, -1)),
        "cusp": s((0, 2, 1), (3, 0, -1)),
        "nodal": s((0, 2, 1), (3, 0, -1), (2, 0, -1)),
        "hyperbola": s((1, 1, 1), (0, 0, -1)),
        # f = s^3 - 2 s + 1 with s = x + y: f_x = f_y, h = f_x, Q = res(1, 1) = 1
        "diagonal": s((3, 0, 1), (2, 1, 3), (1, 2, 3), (0, 3, 1), (1, 0, -2), (0, 1, -2), (0, 0, 1)),
        "lc_x": s((1, 2, 1), (0, 2, 3), (2, 1, -1), (0, 0, 5), (3, 0, 1)),
    }


def teissier() -> list[dict]:
    reqs, meta = [], []
    for c in teissier_curves():
        reqs.append(("curve_q", [curves.make(*c)]))
        meta.append({"curve": list(c)})
    for name, f in special_curves().items():
        reqs.append(("curve_q", [f]))
        meta.append({"name": name, "f": enc_bipoly(f)})
    res = run_batch(reqs)
    rows = []
    for m, r in zip(meta, res):
        row = dict(m)
        if "error" in r:
            row["error"] = r["error"]
        else:
            row["result"], row["h"], row["qsf"] = r["result"], r["h"], r["qsf"]
        row["ref_seconds"] = r["seconds"]
        rows.append(row)
    return rows


def teissier_big(cache_dir: str, cached_only: bool = False) -> list[dict]:
    """Digests of Q = res(f_x, f_y) (h = 1 for these curves) at BASELINE sizes."""
    rows = []
    for (kind, a, b, s) in [("dense", 20, 64, 1), ("sheared", 3, 0, 1)]:
        name = f"{kind}_{a}_{b}_{s}"
        cached = os.path.join(cache_dir, f"outq_{name}.txt")
        prev = {}
        if os.path.exists(os.path.join(GOLD, "teissier_big.jsonl")):
            prev = {tuple(json.loads(l)["curve"]): json.loads(l) for l in open(os.path.join(GOLD, "teissier_big.jsonl"))}
        if os.path.exists(cached) and os.path.getsize(cached) > 0:
            r = json.loads(open(cached).read().splitlines()[0])
        elif (kind, a, b, s) in prev:
            rows.append(prev[(kind, a, b, s)])
            continue
        elif cached_only:
            print(f"skip Q {name}: no cached reference output")
            continue
        else:
            f = curves.make(kind, a, b, s)
            r = run_batch([("resultant_y", [curves.derive_x(f), curves.derive_y(f)])])[0]
        res = r["result"]
        ints = [int(c, 16) for c in res]
        rows.append({"curve": [kind, a, b, s], "deg": len(res) - 1, "max_bits": max(abs(c).bit_length() for c in ints),
                     "sha256": digest(res), "lc": res[-1], "c0": res[0], "ref_seconds": r["seconds"]})
    return rows



def sylvester_acceptance() -> list[dict]:
    """SPEC.md:632 acceptance #2: resultant == Sylvester determinant on >= 500 random pairs,
    deg <= 6, coefficients <= 2^16.  Both sides come from the reference: its resultant
    (elim.cpp:95-136) and its own Bareiss oracle (proj/tests/oracles.cpp:82-120); the fixture
    stores the inputs and the sha256 of the (equal) outputs."""
    rng = random.Random(632)
    pairs = []
    while len(pairs) < 500:
        def one(dmin):
            d = rng.randint(dmin, 6)
            dens = rng.choice((1.0, 0.7, 0.4))
            f = {}
            for i in range(d + 1):
                for j in range(d + 1 - i):
                    if rng.random() <= dens:
                        c = rng.randint(-2**16, 2**16)
                        if c:
                            f[(i, j)] = c
            return f
        p, q = one(1), one(0)
        if not p or not q:  # the Sylvester oracle needs two nonzero inputs (oracles.cpp:86)
            continue
        if rng.random() < 0.25 and p:  # share the Sylvester shape q ~ p_y more often
            q = {(i, j - 1): j * c for (i, j), c in p.items() if j}
            if not q:
                continue
        pairs.append((p, q))
    reqs = []
    for p, q in pairs:
        reqs.append(("resultant_y", [p, q]))
        reqs.append(("sylvester_y", [p, q]))
    out = run_batch(reqs)
    rows = []
    for k, (p, q) in enumerate(pairs):
        r, s_ = out[2 * k], out[2 * k + 1]
        if "error" in r:
            rows.append({"p": enc_bipoly(p), "q": enc_bipoly(q), "error": r["error"]})
            continue
        assert r["result"] == s_["result"], f"reference resultant != Sylvester oracle on pair {k}"
        rows.append({"p": enc_bipoly(p), "q": enc_bipoly(q), "deg": len(r["result"]) - 1,
                     "sha256": digest(r["result"])})
    return rows

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--cache", default=os.path.join(HERE, "_gold_cache"))
    ap.add_argument("--cached-only", action="store_true", help="--big: use only cached reference outputs")
    ap.add_argument("--big-only", action="store_true", help="only rewrite configs_big / teissier_big")
    ap.add_argument("--only", default="", help="rewrite one small fixture (e.g. sylvester_acceptance)")
    args = ap.parse_args()
    if args.only:
        write(f"{args.only}.jsonl", globals()[args.only]())
        return
    if args.big_only:
        write("configs_big.jsonl", configs_big(args.cache, args.cached_only))
        write("teissier_big.jsonl", teissier_big(args.cache, args.cached_only))
        return
    elim = subprocess.run([DRIVER, "elim_cases"], capture_output=True, text=True, check=True).stdout
    write("elim_cases.jsonl", [json.loads(l) for l in elim.splitlines() if l.strip()])
    write("worked.jsonl", worked())
    write("resultant_random.jsonl", resultant_random())
    write("univariate_random.jsonl", univariate_random())
    write("configs_small.jsonl", configs_small())
    write("bivariate_gcd.jsonl", bivariate_gcd())
    write("teissier.jsonl", teissier())
    write("sylvester_acceptance.jsonl", sylvester_acceptance())
    if args.big:
        write("configs_big.jsonl", configs_big(args.cache, args.cached_only))
        write("teissier_big.jsonl", teissier_big(args.cache, args.cached_only))


if __name__ == "__main__":
    main()
