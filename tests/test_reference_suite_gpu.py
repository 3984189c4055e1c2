"""The reference's OWN test binaries, with elim.cpp replaced by the GPU drop-in TU.

oracle/Makefile links each /root/reference/proj/tests/test_*.cpp against the reference
library minus elim.cpp plus paper_1103_4697_b200/cxx/curvetop_elim_gpu.cpp + libctg.so
(oracle/_ref/test_*_gpu).  Every curvetop::resultant / yun_squarefree / gcd_univariate /
square_free_part call those tests make -- directly or through lift / bisolve / realroots /
pipeline helpers -- runs on the GPU.  test_lift is restricted to the cases the reference
itself finishes ("lift_complete: worked examples" stalls off the hot path).
"""

import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")

CASES = [
    ("test_elim_gpu", [], 10, 832),
    ("test_polycore_gpu", [], 13, 997),
    ("test_realroots_gpu", [], 14, 1367),
    ("test_bisolve_gpu", [], 10, 390),
    ("test_lift_gpu", ["-tc=teissier_bound,intermediate_fiber,fast_lift"], 4, 46),
]


@pytest.mark.parametrize("binary,args,cases,checks", CASES, ids=[c[0] for c in CASES])
def test_reference_suite_on_gpu_elim(binary, args, cases, checks):
    path = os.path.join(REF, binary)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle gpu_tests in the build container)")
    r = subprocess.run([path, *args], capture_output=True, text=True, timeout=600)
    summary = r.stdout + r.stderr
    assert r.returncode == 0, summary[-3000:]
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", summary)
    a = re.search(r"assertions: (\d+) \| (\d+) passed \| (\d+) failed", summary)
    assert m and a, summary[-2000:]
    assert (int(m.group(1)), int(m.group(3))) == (cases, 0)
    assert (int(a.group(1)), int(a.group(3))) == (checks, 0)


@pytest.mark.parametrize("binary,args,cases,checks", [c for c in CASES if c[0] in ("test_elim_gpu", "test_bisolve_gpu")],
                         ids=["test_elim_gpu", "test_bisolve_gpu"])
def test_reference_suite_prime_sharded(binary, args, cases, checks):
    """The same reference tests with CTG_DEVICES=0,0,0: every curvetop::resultant the reference's
    callers make runs prime-sharded over three shards (here all on cuda:0: the device-copy
    exchange) through ctg_opts.n_devices -- the multi-GPU product path behind the unchanged API."""
    path = os.path.join(REF, binary)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle gpu_tests in the build container)")
    env = dict(os.environ, CTG_DEVICES="0,0,0")
    r = subprocess.run([path, *args], capture_output=True, text=True, timeout=600, env=env)
    summary = r.stdout + r.stderr
    assert r.returncode == 0, summary[-3000:]
    a = re.search(r"assertions: (\d+) \| (\d+) passed \| (\d+) failed", summary)
    assert a and (int(a.group(1)), int(a.group(3))) == (checks, 0), summary[-2000:]
