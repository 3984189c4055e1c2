"""Loading helpers for the reference-generated fixtures in tests/golden/ (see oracle/make_golden.py)."""

import json
import os

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        return []
    with open(path) as fh:
        return [json.loads(l) for l in fh if l.strip()]


def dec_upoly(hexes):
    return [int(c, 16) for c in hexes]


def dec_bipoly(terms):
    out = {}
    for ex, ey, c in terms:
        out[(ex, ey)] = out.get((ex, ey), 0) + int(c, 16)
    return {k: v for k, v in out.items() if v}


def dec_sqf(r):
    return int(r["unit"], 16), [(dec_upoly(f["poly"]), f["mult"]) for f in r["factors"]]


def dec_arg(a):
    if a and isinstance(a[0], list):
        return dec_bipoly(a)
    return dec_upoly(a)
