#!/usr/bin/env python
"""bench.py -- res(f, f_y) on B200: mod-p resultants/s and wall ms, vs the reference CPU path.

Metric (BASELINE.json): "res(f,f_y) wall ms + mod-p resultants/s at 1/2/4/8 B200 vs host-CPU ref".
  value  = mod-p resultants per second over the whole job, inputs resident in HBM
           (units = P * D per curve: primes x result coefficients);
  e2e    = the same metric through the reference-facing C ABI (ctg_resultant_batch) with HOST
           buffers: H2D of the coefficient limbs, all kernels, D2H of the exact result.
Workload (config.workload): BASELINE.json configs[2], the headline: random dense f of total
degree 30 with 128-bit coefficients (synthetic, the §8(d) generator), 64 curves per step processed
by one batched plan (every kernel launch covers all curves).  configs[1] (d=20 / 64-bit, 256
curves per step) is measured as an extra key ("d20_b64"); one d=30 curve through ctg_resultant
is key "headline".  Every curve whose seed has a reference digest (tests/golden/configs_big.jsonl,
made by the reference itself) is checked against it, outside the timed regions.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--workload d30_b128|d20_b64|...]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N     (prime sharding + NCCL)
  python bench.py --impl reference ...      (the reference CPU implementation, oracle/_ref, all host cores)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "res(f,f_y) wall ms + mod-p resultants/s at 1/2/4/8 B200 vs host-CPU ref"
UNIT = "mod-p resultants/s"
WORKLOADS = {
    # name: (kind, a, b, description, nominal units per curve = P * D for seed 1)
    "d20_b64": ("dense", 20, 64, "random dense f, total degree 20, 64-bit coefficients (BASELINE configs[1])",
                90 * 381),
    "d30_b128": ("dense", 30, 128, "random dense f, total degree 30, 128-bit coefficients (BASELINE configs[2])",
                 259 * 871),
    "d10_b10": ("dense", 10, 10, "random dense f, total degree 10, 10-bit coefficients (BASELINE configs[0])",
                11 * 91),
    "d16_b1024": ("dense", 16, 1024, "random dense f, total degree 16, 1024-bit coefficients (BASELINE configs[4])",
                  1031 * 241),
}
REFDRIVER = os.path.join(REPO, "oracle", "_ref", "refdriver")
# Per-curve units (P * D with P = primes the curve ALONE needs, D = coefficients of its R) for
# seeds 1..n of every workload (scripts/units_table.py): both arms count the same units per
# curve, whatever prime count a batched plan happens to use.
UNITS_FILE = os.path.join(REPO, "bench_units.json")


def curve_units(workload, seeds):
    try:
        with open(UNITS_FILE) as fh:
            table = json.load(fh)[workload]
    except (OSError, KeyError, ValueError):
        return None
    if max(seeds) > len(table):
        return None
    return sum(table[s - 1] for s in seeds)
DEFAULT_BATCH = {"d30_b128": 64, "d20_b64": 256, "d16_b1024": 64, "d10_b10": 64}
GOLDEN_BIG = os.path.join(REPO, "tests", "golden", "configs_big.jsonl")


def workload_config(workload):
    """config of the JSON line: identical in both arms (the workload and the unit of work)."""
    kind, a, b, desc, _ = WORKLOADS[workload]
    return {"workload": desc, "generator": f"{kind}({a}, {b}, seed), SURVEY.md §8(d)",
            "units": "mod-p resultants = P * D per curve, P = primes the curve alone needs (bench_units.json)"}


def golden_digests(workload):
    """{seed: row} of the reference's own digests of res(f, f_y) for this workload."""
    kind, a, b, _, _ = WORKLOADS[workload]
    out = {}
    try:
        with open(GOLDEN_BIG) as fh:
            for line in fh:
                r = json.loads(line)
                if r["curve"][:3] == [kind, a, b]:
                    out[r["curve"][3]] = r
    except OSError:
        pass
    return out


def digest(coeffs):
    import hashlib
    return hashlib.sha256(",".join(format(c, "x") for c in coeffs).encode()).hexdigest()


def check_golden(row, R, what):
    if not (len(R) - 1 == row["deg"] and digest(R) == row["sha256"]):
        raise SystemExit(f"PARITY FAILURE: {what} differs from the reference digest for curve {row['curve']}")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="d30_b128", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0, help="curves per step (seeds 1..B; 0 = workload default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-headline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the d20_b64 extra measurement")
    a = ap.parse_args()
    if a.batch <= 0:
        a.batch = DEFAULT_BATCH[a.workload]
    return a


# ----------------------------------------------------------------------------
# clocks sampled during the timed region
# ----------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation (oracle/_ref), all host cores
# ----------------------------------------------------------------------------
def traffic_for(workload, batch):
    """DRAM bytes (read + write) per K3 launch from one ncu --set full capture of the same
    bench command (profiles/traffic.json, written by scripts/traffic.sh), or None."""
    path = os.path.join(REPO, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh).get(workload)
    except (OSError, ValueError):
        return None
    if not t or t.get("batch") != batch:
        return None
    return t.get("k3_dram_bytes_per_launch")


def run_refdriver(kind, a, b, seed, reps=1, yun=False, timeout=None):
    cmd = [REFDRIVER, "time_res", kind, str(a), str(b), str(seed), str(reps)] + (["yun"] if yun else [])
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


# single-core seconds per curve of the reference on the GPU box's host (r01 measured d20: 10.05 s;
# the others scaled from the build container by the same 2.76x): only used to pick the sample shape
EST_REF_SECONDS = {"d10_b10": 0.008, "d20_b64": 10.0, "d16_b1024": 106.0, "d30_b128": 616.0}


def reference_arm(args):
    """The reference's own CPU implementation of the path (oracle/_ref/refdriver: proj/src/elim.cpp
    compiled unmodified) on every host core, one independent process per curve (the reference is
    single-threaded).  Cheap workloads (d10, d20): K steps of `cores` curves each.  d30/128 needs
    ~10 min per curve, so its bounded sample is ONE wave: min(K, cores) curves (seeds 1..), one
    per core, all started together; value = their units / the wave's wall time."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    kind, a, b, desc, units = WORKLOADS[args.workload]
    if not os.path.exists(REFDRIVER):
        print(json.dumps({"impl": "reference", "unavailable": f"{REFDRIVER} not built (make -C oracle)"}))
        return 0
    cores = os.cpu_count() or 1
    # warm-up: a tiny reference call per step (the CPU has nothing to warm beyond page-in)
    for _ in range(args.warmup):
        run_refdriver("dense", 6, 10, 1)

    def wave(seeds):
        t0 = time.perf_counter()
        procs = [subprocess.Popen([REFDRIVER, "time_res", kind, str(a), str(b), str(s_), "1"],
                                  stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True) for s_ in seeds]
        for p in procs:
            p.wait()
            if p.returncode != 0:
                raise SystemExit(f"reference driver failed (rc {p.returncode})")
        return time.perf_counter() - t0

    one_wave = args.steps * EST_REF_SECONDS[args.workload] > 300
    if one_wave:
        n = max(1, min(args.steps, cores))
        seeds = list(range(1, n + 1))
        total = wave(seeds)
        done_units = curve_units(args.workload, seeds) or units * n
        sample = (f"{n} curves {kind}({a},{b},seed) seeds 1..{n}, one independent process per core, all started "
                  f"together (one wave, {total:.0f} s): curvetop::resultant(f, f_y, Y) from oracle/_ref/refdriver; "
                  f"a step is one curve")
        ms_per_step = 1e3 * total / n
    else:
        walls, done_units = [], 0
        for step in range(args.steps):
            seeds = [1 + (step * cores + c) % 64 for c in range(cores)]
            walls.append(wave(seeds))
            done_units += curve_units(args.workload, seeds) or units * cores
        total = sum(walls)
        sample = (f"{cores} curves per step (one per core, independent processes, seeds 1..64 cycling), "
                  f"curvetop::resultant(f, f_y, Y) from oracle/_ref/refdriver")
        ms_per_step = 1e3 * total / args.steps
    value = done_units / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int (GMP mpz)",
        "data": "synthetic", "config": workload_config(args.workload),
        "sample": {"units_total": done_units, "wall_s": total, "cores": cores},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def main_ours(args):
    import torch

    import paper_1103_4697_b200 as P
    from paper_1103_4697_b200 import curves

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        if os.environ.get("CTG_BENCH_SIM_GLOO") == "1":
            # functional test of the multi-rank path on ONE GPU (ranks share cuda:0, gloo
            # collectives through the host; no kernel waits on another rank): timings are
            # meaningless and not reported as measurements
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    # One explicit (non-default) stream for everything: our kernels, torch fills, NCCL and
    # the timing events.  (Handle 0 would mean "the library's own stream" to libctg.)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    G = world
    peaks = P.microbench_int(dev)
    comm = None
    if world > 1 and os.environ.get("CTG_BENCH_SIM_GLOO") != "1":
        # the library's own NCCL communicator (ctg_comm): residues are exchanged by libctg;
        # torch.distributed only carries the id, the barriers and the max-over-ranks time
        obj = [P.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = P.Comm(world, rank, obj[0], dev)

    m = measure(args, args.workload, args.batch, P, curves, torch, dist, stream, rank, G, peaks, comm)
    line = {
        "metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": G, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32 (31-bit modular, Montgomery)", "data": "synthetic",
        "config": workload_config(args.workload),
        "sample": m["sample"],
        "e2e": m["e2e"],
        "gpu_launches": m["gpu_launches"],
        "roofline": m["roofline"],
        "clocks": m["clocks"],
        "parity": m["parity"],
    }
    if rank == 0 and G == 1 and not args.no_extra and args.workload != "d20_b64":
        x = measure(args, "d20_b64", DEFAULT_BATCH["d20_b64"], P, curves, torch, dist, stream, rank, G, peaks, comm)
        line["d20_b64"] = {"workload": WORKLOADS["d20_b64"][3], "value": x["value"], "unit": UNIT,
                           "ms_per_step": x["ms_per_step"], "sample": x["sample"], "e2e": x["e2e"],
                           "roofline_frac": x["roofline"]["frac"], "stage_ms_per_step": x["roofline"]["stage_ms_per_step"],
                           "gpu_launches": x["gpu_launches"], "clocks": x["clocks"], "parity": x["parity"]}
    if rank == 0 and G == 1 and not args.no_headline:
        line["yun"] = yun_line(P, curves, args.workload)
        line["yun"]["batch"] = yun_batch_line(P, curves, args.workload, args.batch)
    if rank == 0 and G == 1:
        cb = None if args.no_cpu_baseline else cpu_baseline(args.workload, m["units_per_curve"])
        line["cpu_baseline"] = cb
        if not args.no_headline:
            line["headline"] = headline(P, curves, args.workload, cb)
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.barrier()
        if comm:
            comm.close()
        dist.destroy_process_group()
    return 0


def measure(args, workload, B, P, curves, torch, dist, stream, rank, G, peaks, comm=None):
    """One workload: device-resident value (staged events), e2e through the C ABI, K3 roofline,
    and the reference-digest parity of every curve that has one."""
    from paper_1103_4697_b200 import sharding

    dev = torch.cuda.current_device()
    sh = stream.cuda_stream
    assert sh != 0
    kind, a, b, desc, _ = WORKLOADS[workload]
    gold = golden_digests(workload)

    # synthetic curves (seeds 1..B), one batched plan: every launch covers all B curves
    fs = [curves.make(kind, a, b, s) for s in range(1, B + 1)]
    pairs = [(f, curves.derive_y(f)) for f in fs]
    plan = P.Plan(pairs)
    info = plan.info
    Pn, N, D = info["n_primes"], info["n_points"], info["n_coeffs"]
    W = info["out_limbs"] + 1
    # mod-p resultants per step: P * D per curve with the curve's own prime count (the batched
    # plan may use a few more primes, for the largest bound of the batch: not counted)
    units_step = curve_units(workload, range(1, B + 1)) or B * Pn * D
    k0, k1, Pb = sharding.prime_block(Pn, G, rank)  # rows per rank block (uniform for the all-gather)
    j0, j1, Jb = sharding.coeff_block(D, G, rank)
    plan.upload(sh)

    send = torch.zeros((B, Pb, N), dtype=torch.int32, device=dev)
    # G > 1: the column-block exchange -- K4 writes each coefficient by destination rank
    # (ctg_plan_interp_cols: [G][B][Pb][Jc]), one all-to-all, K5 on this rank's columns
    Jc = (D + G - 1) // G
    xsend = torch.zeros((G, B, Pb, Jc), dtype=torch.int32, device=dev) if G > 1 else None
    xrecv = torch.zeros((G, B, Pb, Jc), dtype=torch.int32, device=dev) if G > 1 else None
    out = torch.zeros((B * Jb * W,), dtype=torch.int32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)

    # events: start | K1 reduce | K2 eval | K3 mod-p resultant | K4 interp | exchange | K5 CRT
    STAGES = ("reduce", "eval", "modres", "interp", "exchange", "crt")
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(STAGES) + 1)]
    stage_ms = [0.0] * len(STAGES)

    def crt():
        if G > 1:
            if j1 > j0:
                plan.crt_cols(xrecv.data_ptr(), G, rank, Pb, out.data_ptr(), sh)
        else:
            plan.crt_batch(send.data_ptr(), j0, j1, out.data_ptr(), sh, curve_stride=Pb * N)

    def step(timed=False):
        if timed:
            evs[0].record(stream)
        for i, s_ in enumerate((1, 4, 5, 3)):  # K1, K2, K3 (+ exact fallback), K4
            if s_ == 3 and G > 1:
                plan.interp_cols(k0, k1, send.data_ptr(), G, Pb, xsend.data_ptr(), sh, curve_stride=Pb * N)
            else:
                plan.stage(s_, k0, k1, send.data_ptr(), sh, curve_stride=Pb * N)
            if timed:
                evs[i + 1].record(stream)
        if comm:  # ctg_comm_all_to_all: libctg's NCCL communicator (grouped send / recv), launch stream
            comm.all_to_all(xsend.data_ptr(), xrecv.data_ptr(), xsend[0].numel(), sh)
        elif G > 1:  # CTG_BENCH_SIM_GLOO: functional multi-rank test on one GPU (the all-to-all
            # emulated by an all-gather of the send blocks, this rank's column blocks kept)
            gathered = torch.empty((G,) + tuple(xsend.shape), dtype=xsend.dtype, device=dev)
            dist.all_gather_into_tensor(gathered.view(-1, Pb, Jc), xsend.view(-1, Pb, Jc))
            xrecv.copy_(gathered[:, rank])
        if timed:
            evs[5].record(stream)
        crt()
        if timed:
            evs[6].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    plan.check(sh)
    launches0 = plan.launches

    total_ms = 0.0
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            flush.fill_(1)  # L2 flush between timed iterations (outside the events)
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            step(timed=True)
            torch.cuda.synchronize()
            total_ms += evs[0].elapsed_time(evs[-1])
            for i in range(len(STAGES)):
                stage_ms[i] += evs[i].elapsed_time(evs[i + 1])
    gpu_launches = plan.launches - launches0
    plan.check(sh)
    t_max = total_ms
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    ms_per_step = t_max / args.steps
    value = units_step / (ms_per_step * 1e-3)

    # parity (outside the timed region): the device-resident batch against the reference digests
    parity = {"reference_digests": sorted(s_ for s_ in gold if s_ <= B), "source": "tests/golden/configs_big.jsonl"}
    if G == 1:
        host = out.cpu().numpy().view("uint32").reshape(B, D, W)
        for s_ in parity["reference_digests"]:
            check_golden(gold[s_], plan.decode(host[s_ - 1]), "device-resident batch")
        parity["device_resident"] = "bit-exact"

    # --- e2e through the C ABI with host buffers --------------------------------------
    # G > 1: every rank calls ctg_resultant_batch with ctg_opts.comm (prime-sharded product
    # path: parse + plan + H2D + K1-K4 on its primes + NCCL all-gather + K5 on its coefficient
    # block + all-gather of the limbs + D2H + decode); the time is the max over ranks.
    e2e_phases = None
    hb = P.HostBatch(pairs)
    sim = G > 1 and comm is None  # gloo simulation on one GPU: shards via the device-list path
    kw = {"comm": comm} if comm else ({"devices": [dev] * G} if sim else {})
    for _ in range(max(1, args.warmup)):
        if dist:
            dist.barrier()
        P.resultant_batch_raw(hb, **kw)
    walls = []
    for _ in range(args.steps):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        P.resultant_batch_raw(hb, **kw)
        walls.append(time.perf_counter() - t0)
        st = P.last_call_stats()
        h2d, d2h = st["h2d_bytes"], st["d2h_bytes"]
    e2e_ms = 1e3 * sum(walls) / len(walls)
    if dist:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_phases = {k: st[k] for k in ("setup_ms", "h2d_ms", "device_ms", "d2h_ms", "decode_ms", "total_ms")}
    # parity of the product path (outside the timed region): every reference-pinned seed
    chk = [s_ for s_ in parity["reference_digests"]]
    got = P.resultant_batch([pairs[s_ - 1] for s_ in chk], **kw) if chk else []
    if rank == 0:
        for s_, R in zip(chk, got):
            check_golden(gold[s_], R, "ctg_resultant_batch" + (f" (prime-sharded, G={G})" if G > 1 else ""))
    parity["e2e" if G == 1 else "sharded_e2e"] = "bit-exact"
    e2e_value = units_step / (e2e_ms * 1e-3)

    # --- roofline of the dominant kernel: K3, the mod-p resultant (north_star: >= 50% of IMAD peak)
    n = info["deg_p"]
    sm = {nm: v / args.steps for nm, v in zip(STAGES, stage_ms)}
    units_launch = B * (k1 - k0) * N
    imad_launch = 4.0 * units_launch * (n * n + n - 2)
    achieved = imad_launch / (sm["modres"] * 1e-3) / 1e12
    peak = peaks["imad_per_s"] / 1e12
    roofline = {"bound": "int32-imad", "achieved": achieved, "peak": peak, "unit": "TIMAD/s",
                "frac": achieved / peak, "traffic": traffic_for(workload, B),
                "kernel": f"K3 = k_modres_fast<{n}> (fused division-free Euclid) + k_modres_general (flagged units)",
                "algorithmic": f"4 IMAD x (n^2+n-2) mulmods x {units_launch} units per launch, n={n} (SURVEY §8d)",
                "peak_source": "measured live: ctg_microbench_int (8 IMAD chains/thread, all SMs)",
                "imad_wide_peak_T": peaks["imad_wide_per_s"] / 1e12,
                "mmul2_peak_G": peaks["mmul2_per_s"] / 1e9,
                # K3's count over K2 + K3 time: the evaluation stage charged to the resultant
                "stage2_frac": imad_launch / ((sm["eval"] + sm["modres"]) * 1e-3) / 1e12 / peak,
                "stage_ms_per_step": sm}
    plan.close()
    del send, xsend, xrecv, out, flush
    return {
        "value": value, "ms_per_step": ms_per_step, "units_per_curve": units_step / B,
        "sample": {"curves_per_step": B, "seeds": f"1..{B}", "primes": Pn, "points": N, "coeffs": D,
                   "units_per_step": units_step, "parallelism": f"prime-shard{G}" if G > 1 else "single",
                   "l2": "flushed (256 MB write) between timed steps", "res_ms_per_curve": ms_per_step / B},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "res_ms_per_curve": e2e_ms / B,
                "path": "ctg_resultant_batch (C ABI), host CSR limbs in/out" + (f", ctg_opts.comm over {G} ranks" if G > 1 else ""),
                "phases_ms_last_call": e2e_phases},
        "gpu_launches": int(gpu_launches), "roofline": roofline, "clocks": clk.summary(), "parity": parity,
    }


def headline(P, curves, workload, cb):
    """The north-star config: one d=30 / 128-bit curve through ctg_resultant (host buffers),
    against the reference timed live on one host core in this run (cpu_baseline)."""
    f = curves.make("dense", 30, 128, 1)
    hp, hq = P.HostBipoly(f), P.HostBipoly(curves.derive_y(f))
    for _ in range(3):
        P.resultant_raw(hp, hq)
    ts, dev = [], []
    for _ in range(10):
        t0 = time.perf_counter()
        P.resultant_raw(hp, hq)
        ts.append(1e3 * (time.perf_counter() - t0))
        dev.append(P.last_call_stats()["device_ms"])
    ms = statistics.median(ts)
    out = {"workload": "dense d=30, 128-bit, seed 1 (BASELINE configs[2]), one curve per call", "e2e_ms_median": ms,
           "device_phase_ms_median": statistics.median(dev)}
    if workload == "d30_b128" and cb and cb.get("seconds_per_curve"):
        out["reference_cpu_s"] = cb["seconds_per_curve"]
        out["reference_cpu_source"] = "cpu_baseline of this run (oracle/_ref/refdriver, 1 host core, seed 1)"
        out["speedup_vs_reference_1gpu"] = cb["seconds_per_curve"] * 1e3 / ms
    return out


def yun_line(P, curves, workload):
    """Second §8 row: yun_squarefree(R) through the C ABI for the workload's seed-1 curve
    (and the singular sheared K=3 family, the Yun stress config), GPU wall ms (median of 5).
    "standalone": R from an earlier call (its own K1 + square-freeness probe on the GPU while
    the host takes the content); "after_resultant": right behind ctg_resultant(f, f_y) of the
    same curve, as CurveContext calls it (lift.cpp:64-67: the probe the resultant left behind)."""
    out = {}
    kind, a, b, _, _ = WORKLOADS[workload]
    tiny = curves.make("dense", 8, 10, 1)  # deg R = 56: its call leaves its own probe behind
    for name, (k_, a_, b_) in ((workload, (kind, a, b)), ("sheared_k3", ("sheared", 3, 0))):
        f = curves.make(k_, a_, b_, 1)
        hf, hq = P.HostBipoly(f), P.HostBipoly(curves.derive_y(f))
        R = P.resultant(f, curves.derive_y(f))
        hp = P.HostUpoly(R)
        row = {"deg_R": len(R) - 1, "path": "ctg_yun_squarefree (C ABI), host CSR limbs in/out"}
        for mode in ("standalone", "after_resultant"):
            ts, dev, launches = [], [], []
            for it in range(7):
                if mode == "standalone":
                    P.resultant(tiny, curves.derive_y(tiny))  # the probe cache now holds another R
                else:
                    P.resultant_raw(hf, hq)
                t0 = time.perf_counter()
                fac = P.yun_squarefree_raw(hp)
                if it >= 2:
                    ts.append(1e3 * (time.perf_counter() - t0))
                    st = P.last_call_stats()
                    dev.append(st["device_ms"])
                    launches.append(st["kernel_launches"])
            row[mode] = {"gpu_ms_median": statistics.median(ts), "device_phase_ms_median": statistics.median(dev),
                         "kernel_launches": launches[-1]}
        row["pattern"] = "".join(f"({d})^{m}" for d, m in fac)
        # the standalone call is the headline (no state carried over from the resultant)
        row["gpu_ms_median"] = row["standalone"]["gpu_ms_median"]
        out[name] = row
    out["sheared_k3"]["reference_cpu_s"] = 29.2  # SURVEY §6.2, oracle/_ref in the build container
    return out


def yun_batch_line(P, curves, workload, B):
    """Yun of every R of the workload's batch through ctg_yun_squarefree_batch (CurveContext
    over many curves: one probe launch for all, contents on the host meanwhile)."""
    kind, a, b, _, _ = WORKLOADS[workload]
    pairs = [(f, curves.derive_y(f)) for f in (curves.make(kind, a, b, s) for s in range(1, B + 1))]
    hb = P.HostUpolyBatch(P.resultant_batch(pairs))
    P.yun_squarefree_batch(hb, raw=True)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        pats = P.yun_squarefree_batch(hb, raw=True)
        ts.append(1e3 * (time.perf_counter() - t0))
    ms = statistics.median(ts)
    return {"curves": B, "ms_median": ms, "ms_per_curve": ms / B,
            "path": "ctg_yun_squarefree_batch (C ABI), host CSR limbs in/out",
            "square_free": sum(1 for p in pats if len(p) == 1 and p[0][1] == 1)}


def cpu_baseline(workload, units_per_curve):
    kind, a, b, desc, _ = WORKLOADS[workload]
    if not os.path.exists(REFDRIVER):
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": "oracle/_ref/refdriver not built", "note": "run make -C oracle"}
    try:
        r = run_refdriver(kind, a, b, 1, timeout=1500)
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"failed: {e}"}
    secs = r["res_seconds_best"]
    units_per_curve = curve_units(workload, [1]) or units_per_curve
    return {"value": units_per_curve / secs, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"1 curve {kind}({a},{b},seed=1): curvetop::resultant(f, f_y, Y), 1 thread, {secs:.2f} s",
            "seconds_per_curve": secs}


def main():
    args = parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
