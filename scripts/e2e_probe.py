import time, sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import paper_1103_4697_b200 as P
from paper_1103_4697_b200 import curves
w = sys.argv[1] if len(sys.argv) > 1 else "d30_b128"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
kind, a, b = curves.CONFIGS[w]
pairs = [(f, curves.derive_y(f)) for f in (curves.make(kind, a, b, s) for s in range(1, B + 1))]
hb = P.HostBatch(pairs)
L = P.lib()
for it in range(6):
    outs = (P._UpolyBuf * B)()
    o = P._opts(None)
    t0 = time.perf_counter()
    st = L.ctg_resultant_batch(B, hb.p, hb.q, 0, outs, C.byref(o))
    t1 = time.perf_counter()
    L.ctg_upoly_free_batch(outs, B)
    t2 = time.perf_counter()
    s = P.last_call_stats()
    print(json.dumps({"it": it, "status": st, "call_ms": (t1 - t0) * 1e3, "free_ms": (t2 - t1) * 1e3,
                      "c_total": s["total_ms"], "h2d_ms": s["h2d_ms"], "dev": s["device_ms"], "dec": s["decode_ms"]}))
