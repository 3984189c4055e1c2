"""Device-resident step of the d20 workload (256 curves): one 256-curve plan on one stream vs
C-curve plans rotating over S streams (the batch path's schedule), inputs resident, L2 flushed
between steps; prints ms per step of each schedule."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

B = 256
fs = [curves.make("dense", 20, 64, s) for s in range(1, B + 1)]
pairs = [(f, curves.derive_y(f)) for f in fs]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")


def setup(chunk, nstreams):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    jobs = []
    for c0 in range(0, B, chunk):
        plan = P.Plan(pairs[c0:c0 + chunk])
        info = plan.info
        Pn, N, D, W = info["n_primes"], info["n_points"], info["n_coeffs"], info["out_limbs"] + 1
        st = streams[len(jobs) % nstreams]
        plan.upload(st.cuda_stream)
        rows = torch.zeros((plan.info["batch"], Pn, N), dtype=torch.int32, device="cuda")
        out = torch.zeros((plan.info["batch"] * D * W,), dtype=torch.int32, device="cuda")
        jobs.append((plan, st, rows, out, Pn, N, D))
    torch.cuda.synchronize()
    return streams, jobs


def step(streams, jobs, main):
    ev = torch.cuda.Event()
    ev.record(main)
    for s in streams:
        s.wait_event(ev)
    for plan, st, rows, out, Pn, N, D in jobs:
        sh = st.cuda_stream
        for s_ in (1, 4, 5, 3):
            plan.stage(s_, 0, Pn, rows.data_ptr(), sh, curve_stride=Pn * N)
        plan.crt_batch(rows.data_ptr(), 0, D, out.data_ptr(), sh, curve_stride=Pn * N)
    for s in streams:
        e = torch.cuda.Event()
        e.record(s)
        main.wait_event(e)


main = torch.cuda.current_stream()
for chunk, ns in [(256, 1), (64, 1), (64, 2), (64, 3), (64, 4), (32, 4), (128, 2)]:
    streams, jobs = setup(chunk, ns)
    for _ in range(3):
        step(streams, jobs, main)
    torch.cuda.synchronize()
    t = 0.0
    for _ in range(10):
        flush.fill_(1)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        step(streams, jobs, main)
        b.record(main)
        torch.cuda.synchronize()
        t += a.elapsed_time(b)
    print(f"chunk {chunk:3d} streams {ns}: {t / 10:.3f} ms per 256-curve step", flush=True)
