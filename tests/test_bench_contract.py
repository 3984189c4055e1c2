"""bench.py's reference arm on the CPU (the reference compiled unmodified in oracle/_ref, run
on every host core): the JSON line must follow the driver contract for `--impl reference`.
Skipped when the reference driver has not been built (make -C oracle)."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(os.path.join(REPO, "oracle", "_ref", "refdriver")),
                    reason="oracle/_ref/refdriver not built")
def test_reference_arm_json_contract():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--workload",
                          "d10_b10", "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300,
                         cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["value"] > 0 and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    # units per step come from the shared per-curve table (bench_units.json), as in our arm
    assert line["sample"]["units_total"] > 0 and line["config"]["workload"]
