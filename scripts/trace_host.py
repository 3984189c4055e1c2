"""Host-side phase trace of ctg_resultant_batch (CTG_TRACE_HOST=1): where the e2e time goes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CTG_TRACE_HOST"] = "1"
import paper_1103_4697_b200 as P
from paper_1103_4697_b200 import curves
wl = sys.argv[1] if len(sys.argv) > 1 else "dense 20 64"
kind, d, bits = wl.split()
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
fs = [curves.make(kind, int(d), int(bits), s) for s in range(1, B + 1)]
hb = P.HostBatch([(f, curves.derive_y(f)) for f in fs])
for i in range(6):
    t = time.perf_counter()
    P.resultant_batch_raw(hb)
    w = time.perf_counter() - t
    st = P.last_call_stats()
    print(f"wall {w*1e3:.3f} ms", {k: round(st[k], 3) for k in ("setup_ms", "h2d_ms", "device_ms", "decode_ms", "total_ms")}, flush=True)
