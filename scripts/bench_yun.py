"""Time yun_squarefree / square_free_part on the GPU for R = res(f, f_y) of the BASELINE configs.

Prints one JSON line per config: GPU wall ms (C-ABI call, host buffers) and the reference's
CPU time where it is known (SURVEY.md §6.2 / oracle/_ref runs)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

REF_YUN_S = {"d10_b10": 1.21, "sheared_k2": 2.11, "sheared_k3": 29.2, "d20_b64": 5000.0, "d30_b128": 3.0e5,
             "d16_b1024": 2.2e4}  # SURVEY §6.2 (d>=20: extrapolated, "> budget")

for name in ["d10_b10", "sheared_k2", "sheared_k3", "d20_b64", "d16_b1024", "d30_b128"]:
    kind, a, b = curves.CONFIGS[name]
    f = curves.make(kind, a, b, 1)
    R = P.resultant(f, curves.derive_y(f))
    hp = P.HostUpoly(R)
    for _ in range(2):
        P.yun_squarefree(R)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        unit, fac = P.yun_squarefree(R)
        ts.append(1e3 * (time.perf_counter() - t0))
    st = P.last_call_stats()
    pattern = "".join(f"({len(p) - 1})^{m}" for p, m in fac)
    t1 = time.perf_counter()
    S = P.square_free_part(R)
    sq_ms = 1e3 * (time.perf_counter() - t1)
    print(json.dumps({"config": name, "deg_R": len(R) - 1, "yun_ms_median": statistics.median(ts),
                      "pattern": pattern, "kernel_launches": st["kernel_launches"], "c_phases_ms": {k: round(st[k], 3) for k in ("setup_ms", "device_ms", "decode_ms", "total_ms")}, "sqfp_ms": sq_ms,
                      "ref_cpu_yun_s": REF_YUN_S[name]}), flush=True)
