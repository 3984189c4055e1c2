"""The formal-degree path beyond the fast kernel's deg_y 40 (k_modres_warp, warp per unit):
throughput of dense curves of total degree 40 (fast kernel) vs 41, 50, 64 (k_modres_mw: four units per warp),
16-bit coefficients, 8 curves per call through ctg_resultant_batch (host buffers)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

for d in (40, 41, 50, 64):
    pairs = [(f, curves.derive_y(f)) for f in (curves.dense(d, 16, s) for s in range(1, 9))]
    hb = P.HostBatch(pairs)
    P.resultant_batch_raw(hb)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        P.resultant_batch_raw(hb)
        ts.append(time.perf_counter() - t0)
    st = P.last_call_stats()
    units = st["n_primes"] * st["n_coeffs"] * len(pairs)
    ms = 1e3 * statistics.median(ts)
    print(json.dumps({"deg": d, "kernel": "k_modres_fast" if d <= 40 else "k_eval_ntt + k_modres_mw", "curves": len(pairs),
                      "primes": st["n_primes"], "coeffs": st["n_coeffs"], "ms_per_call": ms,
                      "units_per_s": units / (ms * 1e-3)}))
