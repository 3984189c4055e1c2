"""CPU (gloo, world size 2) test of the prime-sharded exchange used on multiple B200s.

The GPU stages are replaced by their mathematical specification so the multi-rank host
logic can run without GPUs: a rank's residue rows are R mod p_k (from the CPU oracle's exact
R) and its CRT block is a Garner reconstruction over the all-gathered buffer, addressed
exactly as ctg_plan_crt_batch addresses it (paper_1103_4697_b200/sharding.py).  What is
checked: every prime row is produced once, the all-gather layout and the rank-block
addressing agree, and the coefficient blocks reassemble bit-exactly on rank 0.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import curvetop_oracle as O
from paper_1103_4697_b200 import curves, sharding

def _primes(count):
    out, p = [], (1 << 31) - 1
    while len(out) < count:
        if all(p % d for d in range(3, int(p ** 0.5) + 1, 2)):
            out.append(p)
        p -= 2
    return out


def _crt_symmetric(residues, primes):
    x, m = 0, 1
    for r, p in zip(residues, primes):
        t = ((r - x) * pow(m, -1, p)) % p
        x += m * t
        m *= p
    return x - m if x > m // 2 else x


def _worker(rank, world, port, B, result_file):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fs = [curves.dense(5, 12, s) for s in range(1, B + 1)]
    Rs = [O.resultant(f, O.derive_y(f)) for f in fs]
    D = max(len(R) for R in Rs) + 3                      # a degree bound above the true degree
    bound = max(max(abs(c) for c in R) for R in Rs)
    P = 1
    while True:
        primes = _primes(P)
        if np.prod([float(p) for p in primes]) > 4 * float(bound):
            break
        P += 1
    N = D + 5                                            # row pitch (NTT size) >= D
    k0, k1, Pb = sharding.prime_block(P, world, rank)
    # "K1-K4": this rank's rows, layout [B][Pb][N]
    send = torch.zeros((B, Pb, N), dtype=torch.int64)
    for b, R in enumerate(Rs):
        for k in range(k0, k1):
            p = primes[k]
            send[b, k - k0, :len(R)] = torch.tensor([c % p for c in R], dtype=torch.int64)
    parts = [torch.zeros_like(send) for _ in range(world)]
    dist.all_gather(parts, send)
    full = torch.stack(parts).reshape(-1).numpy()        # [G][B][Pb][N]
    # "K5": CRT of this rank's coefficient block through the documented addressing
    j0, j1, Jb = sharding.coeff_block(D, world, rank)
    W = 1
    out = torch.zeros((B * Jb * W,), dtype=torch.int64)
    vals = {}
    for b in range(B):
        for j in range(j0, j1):
            res = [int(full[sharding.row_offset(b, k, B, Pb, N) + j]) for k in range(P)]
            vals[(b, j)] = _crt_symmetric(res, primes)
    gathered = [None] * world
    dist.all_gather_object(gathered, vals)
    if rank == 0:
        merged = {}
        for g in gathered:
            merged.update(g)
        ok = all(merged[(b, j)] == (Rs[b][j] if j < len(Rs[b]) else 0) for b in range(B) for j in range(D))
        ok &= len(merged) == B * D
        # the numeric reassembly helper on a dense [G][B*Jr*W] layout
        dense = np.zeros((world, B * Jb * W), dtype=object)
        for r in range(world):
            a0, a1, _ = sharding.coeff_block(D, world, r)
            Jr = a1 - a0
            blk = np.array([[merged[(b, j)] for j in range(a0, a1)] for b in range(B)], dtype=object)
            dense[r, :B * Jr * W] = blk.reshape(-1)
        re = sharding.reassemble(dense, B, D, W, world)
        ok &= all(int(re[b, j, 0]) == merged[(b, j)] for b in range(B) for j in range(D))
        with open(result_file, "w") as fh:
            fh.write("ok" if ok else "mismatch")
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2])
def test_prime_sharded_exchange_gloo(tmp_path, world):
    result = tmp_path / "result.txt"
    mp.spawn(_worker, args=(world, _free_port(), 3, str(result)), nprocs=world, join=True)
    assert result.read_text() == "ok"


def test_layout_helpers():
    P, G, N, B = 261, 8, 896, 4
    seen = []
    for r in range(G):
        k0, k1, Pb = sharding.prime_block(P, G, r)
        seen += list(range(k0, k1))
        assert Pb == 33
    assert seen == list(range(P))
    offs = {sharding.row_offset(b, k, B, 33, N) for b in range(B) for k in range(P)}
    assert len(offs) == B * P and all(o % N == 0 for o in offs)
    D = 871
    cov = []
    for r in range(G):
        j0, j1, _ = sharding.coeff_block(D, G, r)
        cov += list(range(j0, j1))
    assert cov == list(range(D))
