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
