"""CurveContext's two calls through the C ABI back to back (lift.cpp:64-67): ctg_resultant(f, f_y)
then ctg_yun_squarefree(R) -- C-side phases of each (the Yun call reuses the probe the
resultant left behind when its input is exactly R)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

for (k, a, b) in [("dense", 20, 64), ("dense", 30, 128), ("dense", 16, 1024), ("sheared", 3, 0)]:
    f = curves.make(k, a, b, 1)
    hp, hq = P.HostBipoly(f), P.HostBipoly(curves.derive_y(f))
    R = P.resultant(f, curves.derive_y(f))
    hr = P.HostUpoly(R)
    rs, ys = [], []
    for _ in range(12):
        P.resultant_raw(hp, hq)
        rs.append(P.last_call_stats()["total_ms"])
        P.yun_squarefree_raw(hr)
        ys.append(P.last_call_stats())
    print(json.dumps({"curve": [k, a, b], "resultant_ms": statistics.median(rs),
                      "yun_total_ms": statistics.median(s["total_ms"] for s in ys),
                      "yun_setup_ms": statistics.median(s["setup_ms"] for s in ys),
                      "yun_device_ms": statistics.median(s["device_ms"] for s in ys),
                      "yun_launches": ys[-1]["kernel_launches"]}))
