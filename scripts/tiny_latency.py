"""Latency of the drop-in's small calls (realroots.cpp:119,136,196 and lift.cpp:155 call
gcd_univariate on tiny polynomials): C-side total / device ms per call through the C ABI."""
import json
import os
import random
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402

rng = random.Random(5)
for deg in (2, 5, 10, 20, 50, 100):
    a = [rng.randint(-50, 50) for _ in range(deg)] + [1]
    b = [rng.randint(-50, 50) for _ in range(deg - 1)] + [3]
    ha, hb = P.HostUpoly(a), P.HostUpoly(b)
    for _ in range(20):
        P.gcd_univariate(a, b)
    ts, st = [], []
    for _ in range(200):
        t0 = time.perf_counter()
        P.gcd_univariate(a, b)
        ts.append(1e6 * (time.perf_counter() - t0))
        st.append(P.last_call_stats())
    med = {k: statistics.median(s[k] for s in st) * 1e3 for k in ("setup_ms", "device_ms", "decode_ms", "total_ms")}
    print(json.dumps({"op": "gcd_univariate", "deg": deg, "python_call_us": statistics.median(ts),
                      **{k.replace("_ms", "_us"): v for k, v in med.items()},
                      "launches": st[-1]["kernel_launches"]}))
