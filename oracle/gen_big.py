"""TEST INFRASTRUCTURE ONLY: run the reference (oracle/_ref/refdriver) on the full-size
BASELINE curves in parallel and cache its raw outputs for ``make_golden.py --big``.

Each job is one curve: ``res(f, f_y, y)`` through the reference's own ``resultant``
(elim.cpp:95-136) and, where the reference finishes in reasonable time (sheared family,
SURVEY.md §6.2), its ``yun_squarefree`` (elim.cpp:138-165).  Output per curve:
``<cache>/out_<name>.txt`` (first line = refdriver's JSON for the resultant, second line =
Yun when requested).  Longest jobs are started first.

    python oracle/gen_big.py --jobs 6                 # the default seed plan below
    python oracle/make_golden.py --big --cached-only   # fold the cache into tests/golden/
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import make_golden as mg  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

# (kind, a, b, seed, with_yun, est_seconds)   est = build-container seconds per curve
PLAN = ([("dense", 30, 128, s, False, 1700) for s in range(2, 65)]
        + [("dense", 16, 1024, s, False, 290) for s in range(2, 9)]
        + [("dense", 20, 64, s, False, 28) for s in range(2, 65)]
        + [("sheared", 3, 0, s, True, 35) for s in range(2, 6)]
        + [("sheared", 2, 0, s, True, 3) for s in range(3, 6)])


def cache_name(kind: str, a: int, b: int, s: int) -> str:
    return f"{kind}_{a}_{b}_{s}" if kind == "dense" else f"{kind}_{a}_{s}"


def run_one(cache: str, kind: str, a: int, b: int, s: int, with_yun: bool) -> str:
    name = cache_name(kind, a, b, s)
    path = os.path.join(cache, f"out_{name}.txt")
    if os.path.exists(path) and os.path.getsize(path) > 0:
        return f"{name}: cached"
    f = curves.make(kind, a, b, s)
    t0 = time.time()
    r = mg.run_batch([("resultant_fy", [f])])[0]
    lines = [json.dumps(r)]
    if with_yun:
        y = mg.run_batch([("yun", [[int(c, 16) for c in r["result"]]])])[0]
        lines.append(json.dumps(y))
    tmp = path + ".tmp"
    with open(tmp, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    os.replace(tmp, path)
    return f"{name}: {time.time() - t0:.1f} s"


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--cache", default=os.path.join(HERE, "_gold_cache"))
    ap.add_argument("--jobs", type=int, default=max(1, (os.cpu_count() or 2) - 2))
    args = ap.parse_args()
    os.makedirs(args.cache, exist_ok=True)
    plan = sorted(PLAN, key=lambda t: -t[5])
    with cf.ThreadPoolExecutor(args.jobs) as ex:
        futs = [ex.submit(run_one, args.cache, k, a, b, s, y) for (k, a, b, s, y, _) in plan]
        for fu in cf.as_completed(futs):
            print(fu.result(), flush=True)


if __name__ == "__main__":
    main()
