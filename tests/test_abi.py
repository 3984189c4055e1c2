"""CPU checks of the drop-in boundary: libctg.so loads, exports every symbol
include/ctg.h declares, and fails loudly (no CPU fallback) without a device."""

import os
import re

import pytest

import paper_1103_4697_b200 as P

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(REPO, "include", "ctg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ctg_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = P.lib()
    declared = _header_functions()
    assert len(declared) >= 15
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert set(declared) == set(P.EXPORTS)
    assert L.ctg_abi_version() == 2


def test_conventions_without_computation():
    with pytest.raises(P.PreconditionError):
        P.resultant({}, {})


@pytest.mark.skipif(P.device_count() > 0, reason="GPU present")
def test_no_cpu_fallback():
    with pytest.raises(P.CudaError):
        P.resultant({(0, 2): 1, (1, 0): -1}, {(0, 1): 2})


@pytest.mark.skipif(P.device_count() > 0, reason="GPU present")
def test_no_cpu_fallback_any_entry_point():
    """Every compute entry point -- including the r2 batch, device-list and communicator paths --
    raises CudaError on a machine without a GPU instead of computing on the CPU."""
    f = {(0, 2): 1, (1, 0): -1}
    fy = {(0, 1): 2}
    for call in (lambda: P.yun_squarefree([1, 0, -2, 0, 1]),
                 lambda: P.yun_squarefree_batch([[1, 0, -2, 0, 1], [-2, 0, 1]]),
                 lambda: P.gcd_univariate([-1, 0, 1], [-1, 1]),
                 lambda: P.square_free_part([1, 2, 1]),
                 lambda: P.gcd_bivariate(f, fy),
                 lambda: P.resultant_batch([(f, fy)] * 3),
                 lambda: P.resultant_batch([(f, fy)] * 3, devices=[0, 0])):
        with pytest.raises(P.CudaError):
            call()


def test_opts_layout_matches_header():
    """ctg_opts is 32 bytes in both the header (int32 device, verify, n_devices, reserved0,
    pointer devices, pointer comm) and the ctypes mirror."""
    import ctypes
    assert ctypes.sizeof(P._Opts) == 32
    assert P._Opts.devices.offset == 16 and P._Opts.comm.offset == 24
