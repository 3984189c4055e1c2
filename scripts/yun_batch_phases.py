"""ctg_yun_squarefree_batch on the R of the d30 bench batch: C-side phases (setup = contents on
the host while the GPU probes, device = the probe's remaining wait, decode = outputs)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
pairs = [(f, curves.derive_y(f)) for f in (curves.make("dense", 30, 128, s) for s in range(1, B + 1))]
hb = P.HostUpolyBatch(P.resultant_batch(pairs))
P.yun_squarefree_batch(hb, raw=True)
ts, st = [], []
for _ in range(5):
    t0 = time.perf_counter()
    P.yun_squarefree_batch(hb, raw=True)
    ts.append(1e3 * (time.perf_counter() - t0))
    st.append(P.last_call_stats())
print(json.dumps({"curves": B, "wall_ms": statistics.median(ts),
                  **{k: statistics.median(s[k] for s in st) for k in ("setup_ms", "h2d_ms", "device_ms", "decode_ms", "total_ms")},
                  "launches": st[-1]["kernel_launches"]}))
