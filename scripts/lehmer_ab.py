"""A/B of K6's remainder-sequence kernels through ctg_modp_gcd_degree: blocked Lehmer (method 0)
vs one pass per step (method 1) on deg-n square-free inputs (gcd(f, f'), the probe's case).

    python scripts/lehmer_ab.py [n ...]          # kernel ms per method (median of 5)
"""
import random
import statistics
import sys

import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402


def main():
    ns = [int(a) for a in sys.argv[1:]] or [100, 300, 870, 2000, 4000]
    p = P.uni_prime(0, device=0)
    rng = random.Random(1)
    for n in ns:
        f = [rng.randrange(p) for _ in range(n)] + [1]
        df = [(i * f[i]) % p for i in range(1, n + 1)]
        row = {}
        for m in (0, 1, 2):
            ts = [P.modp_gcd_degree(f, df, 0, m, device=0) for _ in range(5)]
            assert len({t["deg"] for t in ts}) == 1
            row[m] = (statistics.median(t["ms"] for t in ts), ts[0]["deg"])
        print(f"n={n}: lehmer {row[0][0]*1e3:.1f} us, per-step {row[1][0]*1e3:.1f} us, "
              f"lehmer small-prime {row[2][0]*1e3:.1f} us (deg {row[0][1]})", flush=True)


if __name__ == "__main__":
    main()
