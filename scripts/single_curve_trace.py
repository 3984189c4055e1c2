"""One d30/128 curve through ctg_resultant (host buffers), CTG_TRACE_HOST breakdown."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

f = curves.make("dense", 30, 128, 1)
hp, hq = P.HostBipoly(f), P.HostBipoly(curves.derive_y(f))
for _ in range(5):
    P.resultant_raw(hp, hq)
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    P.resultant_raw(hp, hq)
    ts.append(1e3 * (time.perf_counter() - t0))
print("e2e ms median", statistics.median(ts), P.last_call_stats(), file=sys.stderr)
