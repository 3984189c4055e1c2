"""Yun through the C ABI at the dense configs: C-side phases (setup / device / decode) and wall ms."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

CASES = [("dense", 20, 64), ("dense", 30, 128), ("dense", 16, 1024), ("sheared", 3, 0)]
RS = {c: P.resultant(curves.make(*c, 1), curves.derive_y(curves.make(*c, 1))) for c in CASES}
# a last small resultant: the single-curve probe cache then holds none of the R below, so
# every Yun call runs standalone (its own K1 + probe); scripts/ctx_phases.py times the cached path
P.resultant(curves.make("dense", 6, 10, 1), curves.derive_y(curves.make("dense", 6, 10, 1)))
for (k, a, b) in CASES:
    R = RS[(k, a, b)]
    hp = P.HostUpoly(R)
    for _ in range(3):
        P.yun_squarefree_raw(hp)
    ts, st = [], []
    for _ in range(10):
        t0 = time.perf_counter()
        P.yun_squarefree_raw(hp)
        ts.append(1e3 * (time.perf_counter() - t0))
        st.append(P.last_call_stats())
    med = {key: statistics.median(s[key] for s in st) for key in ("setup_ms", "h2d_ms", "device_ms", "decode_ms", "total_ms")}
    print(json.dumps({"curve": [k, a, b], "deg": len(R) - 1, "wall_ms": statistics.median(ts), **med,
                      "launches": st[-1]["kernel_launches"], "h2d_bytes": st[-1]["h2d_bytes"]}))
