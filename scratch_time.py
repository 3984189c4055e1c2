import time, json, sys
import paper_1103_4697_b200 as P
from paper_1103_4697_b200 import curves
for name in ["d10_b10", "d20_b64", "d30_b128", "sheared_k3", "d16_b1024"]:
    kind, a, b = curves.CONFIGS[name]
    f = curves.make(kind, a, b, 1); fy = curves.derive_y(f)
    hp, hq = P.HostBipoly(f), P.HostBipoly(fy)
    for it in range(4):
        t = time.perf_counter(); R = P.resultant_host(hp, hq); dt = time.perf_counter() - t
    st = P.last_call_stats()
    print(name, f"{dt*1e3:.2f} ms", len(R)-1, max(abs(c).bit_length() for c in R), json.dumps(st), flush=True)
