import time, sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1103_4697_b200 as P
from paper_1103_4697_b200 import curves
B = 64
fs = [curves.make("dense", 20, 64, s) for s in range(1, B + 1)]
plan = P.Plan([(f, curves.derive_y(f)) for f in fs])
info = plan.info
Pn, N, D, W = info["n_primes"], info["n_points"], info["n_coeffs"], info["out_limbs"] + 1
st = torch.cuda.Stream(); torch.cuda.set_stream(st); sh = st.cuda_stream
plan.upload(sh)
send = torch.zeros((B, Pn, N), dtype=torch.int32, device="cuda")
out = torch.zeros((B * D * W,), dtype=torch.int32, device="cuda")
def step():
    ts = []
    for s_ in (1, 2, 3):
        t = time.perf_counter(); plan.stage(s_, 0, Pn, send.data_ptr(), sh, curve_stride=Pn * N); ts.append(time.perf_counter() - t)
    t = time.perf_counter(); plan.crt_batch(send.data_ptr(), 0, D, out.data_ptr(), sh, curve_stride=Pn * N); ts.append(time.perf_counter() - t)
    return ts
for _ in range(3): step()
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter(); ts = step(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(json.dumps({"host_calls_us": [round(x * 1e6, 1) for x in ts], "enqueue_us": round((t1 - t0) * 1e6, 1), "total_us": round((t2 - t0) * 1e6, 1)}))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st); step(); e1.record(st); torch.cuda.synchronize(); print("gpu_ms", e0.elapsed_time(e1))
