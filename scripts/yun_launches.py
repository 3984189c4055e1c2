"""Yun of the d30/128 resultant three times (for an ncu launch list of the univariate kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1103_4697_b200 as P  # noqa: E402
from paper_1103_4697_b200 import curves  # noqa: E402

f = curves.make("dense", 30, 128, 1)
R = P.resultant(f, curves.derive_y(f))
hp = P.HostUpoly(R)
for _ in range(3):
    P.yun_squarefree_raw(hp)
