"""CTG_TRACE_HOST timeline of one ctg_resultant_batch call (the bench's e2e step)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

kind, a, b, B = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
pairs = [(f, curves.derive_y(f)) for f in (curves.make(kind, a, b, s) for s in range(1, B + 1))]
hb = P.HostBatch(pairs)
for _ in range(3):
    P.resultant_batch_raw(hb)
t0 = time.perf_counter()
P.resultant_batch_raw(hb)
print("wall ms", 1e3 * (time.perf_counter() - t0), P.last_call_stats(), file=sys.stderr)
