"""Wall time of the reference's own test binaries on the reference elim.cpp (oracle/_ref/test_X)
and on the GPU drop-in TU (oracle/_ref/test_X_gpu): the small-input latency of the drop-in
(realroots.cpp:119,136,196 and lift.cpp:155 call gcd_univariate on tiny polynomials)."""
import json
import os
import subprocess
import sys
import time

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
CASES = [("test_realroots", []), ("test_elim", []), ("test_polycore", []), ("test_bisolve", []),
         ("test_lift", ["-tc=teissier_bound,intermediate_fiber,fast_lift"])]  # the rest of test_lift stalls on the reference
for name, args in CASES:
    row = {"test": name, "args": args}
    for tag, exe in (("reference_s", name), ("gpu_dropin_s", name + "_gpu")):
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            r = subprocess.run([os.path.join(REF, exe)] + args, capture_output=True, text=True, timeout=600)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
            row[tag.replace("_s", "_rc")] = r.returncode
            tail = (r.stdout.strip().splitlines() or [""])[-1]
            row[tag.replace("_s", "_summary")] = tail[:120]
        row[tag] = best
    print(json.dumps(row), flush=True)
