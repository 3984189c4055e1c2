"""The synthetic workload generator (paper_1103_4697_b200/curves.py) is
bit-identical to the reference-side generator in oracle/_ref/refdriver (`gen`): the GPU path
and the reference time and check exactly the same curves.  CPU only; skipped when the
reference driver has not been built (make -C oracle)."""

import os
import subprocess

import pytest

from paper_1103_4697_b200 import curves

REFDRIVER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "refdriver")


def _gen(*args):
    out = subprocess.run([REFDRIVER, "gen", *map(str, args)], capture_output=True, text=True, check=True).stdout
    lines = out.split("\n")
    n = int(lines[0].split()[1])
    f = {}
    for ln in lines[1:1 + n]:
        dx, dy, h = ln.split()
        f[(int(dx), int(dy))] = int(h, 16)
    return f


@pytest.mark.skipif(not os.path.exists(REFDRIVER), reason="oracle/_ref/refdriver not built")
@pytest.mark.parametrize("args", [("dense", 3, 40, 7), ("dense", 10, 10, 1), ("dense", 20, 64, 5), ("dense", 30, 128, 64),
                                  ("dense", 16, 1024, 2), ("sheared", 2, 1), ("sheared", 3, 4)])
def test_generator_matches_reference_driver(args):
    want = _gen(*args)
    if args[0] == "dense":
        got = curves.make("dense", args[1], args[2], args[3])
    else:
        got = curves.make("sheared", args[1], 0, args[2])
    assert got == want
