"""Prime sharding across GPUs: layout math and the exchange step.

Every rank owns a contiguous block of the plan's primes and computes those rows of the
residue matrix (K1-K4, no communication).  One all-gather assembles the matrix in the
layout ``[G][B][Pb][N]`` (rank block, curve, row within block, point); each rank then
reconstructs a contiguous block of coefficients (K5) and a second all-gather brings the
exact limbs to rank 0.  The CRT kernels address row ``k`` of curve ``b`` in that buffer as

    (k // Pb) * block_stride + b * curve_stride + (k % Pb) * N,
    block_stride = B * Pb * N,  curve_stride = Pb * N,

which is exactly ``ctg_plan_crt_batch(plan, full, curve_stride, Pb, block_stride, ...)``.
The same helpers drive bench.py on NCCL and tests/test_sharding.py on gloo (CPU).
"""

from __future__ import annotations

import numpy as np


def prime_block(P: int, G: int, rank: int):
    """Rows [k0, k1) of rank `rank` and the uniform block size Pb (last blocks may be short)."""
    Pb = (P + G - 1) // G
    return min(rank * Pb, P), min((rank + 1) * Pb, P), Pb


def coeff_block(D: int, G: int, rank: int):
    """Coefficients [j0, j1) reconstructed by rank `rank` and the uniform block size Jb."""
    Jb = (D + G - 1) // G
    return min(rank * Jb, D), min((rank + 1) * Jb, D), Jb


def strides(B: int, Pb: int, N: int):
    """(curve_stride, block_stride) of the all-gathered residue buffer [G][B][Pb][N] (words)."""
    return Pb * N, B * Pb * N


def row_offset(b: int, k: int, B: int, Pb: int, N: int) -> int:
    curve_stride, block_stride = strides(B, Pb, N)
    return (k // Pb) * block_stride + b * curve_stride + (k % Pb) * N


def reassemble(gathered: np.ndarray, B: int, D: int, W: int, G: int) -> np.ndarray:
    """Per-rank CRT outputs gathered as [G][>= B*Jr*W] words -> [B][D][W] (rank r holds
    coefficients [j0_r, j1_r) of every curve, dense [B][Jr][W])."""
    blocks = []
    for r in range(G):
        j0, j1, _ = coeff_block(D, G, r)
        Jr = j1 - j0
        blocks.append(np.asarray(gathered[r]).reshape(-1)[:B * Jr * W].reshape(B, Jr, W))
    return np.concatenate(blocks, axis=1)
