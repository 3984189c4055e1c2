"""Yun through the C ABI at the dense configs: C-side phases (setup / device / decode) and wall ms."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

for (k, a, b) in [("dense", 20, 64), ("dense", 30, 128), ("dense", 16, 1024), ("sheared", 3, 0)]:
    f = curves.make(k, a, b, 1)
    R = P.resultant(f, curves.derive_y(f))
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
