"""bench.py's multi-rank path (prime sharding, all-gather, rank-block CRT, rank-0 decode and
its exactness check against the one-shot call) run as 2 torchrun ranks sharing cuda:0 with gloo
collectives (CTG_BENCH_SIM_GLOO=1): a functional test of the code the driver runs on N GPUs
with NCCL.  No rank's kernel waits on another rank; the timings are not measurements."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_rank_prime_sharded_bench():
    env = dict(os.environ, CTG_BENCH_SIM_GLOO="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29531", os.path.join(REPO, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--batch", "16"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["sample"]["parallelism"] == "prime-shard2"
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
