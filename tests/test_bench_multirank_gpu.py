"""bench.py's multi-rank path run as 2 torchrun ranks sharing cuda:0 (CTG_BENCH_SIM_GLOO=1):
the device-resident staged step with gloo collectives, and the e2e through ctg_resultant_batch's
prime-sharded product path (device-list mode: both shards on cuda:0, exchange by device copies;
on N real GPUs bench.py passes a ctg_comm and libctg's NCCL does the exchange).  The reference
digest of seed 1 is checked inside bench.py.  No rank's kernel waits on another rank; the
timings are not measurements."""

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
    assert line["parity"]["sharded_e2e"] == "bit-exact" and 1 in line["parity"]["reference_digests"]
