"""A/B of the prime-sharded exchange on one GPU (shards sharing it): "fused" (K4 stores each
coefficient into the owning shard's receive block) vs "copy" (all-gather of whole residue rows by
device copies).  ctg_resultant_batch wall ms through raw host buffers (median of 5), 64 dense
d20/64 curves; G = 1 is the plain single-device call."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

pairs = [(f, curves.derive_y(f)) for f in (curves.make("dense", 20, 64, s) for s in range(1, 65))]
ref = P.resultant_batch(pairs)
hb = P.HostBatch(pairs)


def wall(**kw):
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        P.resultant_batch_raw(hb, **kw)
        ts.append(1e3 * (time.perf_counter() - t0))
    return statistics.median(ts[2:])


print(f"G=1: {wall():.3f} ms", flush=True)
for G in (2, 4, 8):
    for mode in ("fused", "copy"):
        os.environ["CTG_SHARD_EXCHANGE"] = mode
        assert P.resultant_batch(pairs, devices=[0] * G) == ref
        print(f"G={G} {mode}: {wall(devices=[0] * G):.3f} ms", flush=True)
