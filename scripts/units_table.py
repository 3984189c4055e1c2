"""Per-curve unit counts (mod-p resultants = P * D) of the bench workloads:
P = primes the curve alone needs (its own Hadamard bound), D = coefficients of its R.
Printed as the UNITS table bench.py uses for both arms (run once on a GPU box)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

out = {}
for name, (kind, a, b, n) in {"d20_b64": ("dense", 20, 64, 256), "d30_b128": ("dense", 30, 128, 64),
                              "d16_b1024": ("dense", 16, 1024, 64), "d10_b10": ("dense", 10, 10, 64)}.items():
    units = []
    for s in range(1, n + 1):
        f = curves.make(kind, a, b, s)
        info = P.Plan(f, curves.derive_y(f)).info
        units.append(info["n_primes"] * info["n_coeffs"])
    out[name] = units
print(json.dumps(out))
