"""Prime sharding on the real kernels, with G ranks simulated on ONE GPU.

Each simulated rank runs K1-K4 of its prime block into its own [B][Pb][N] buffer (exactly
the bench.py --gpus G path), the buffers are concatenated as the NCCL all-gather would
([G][B][Pb][N]), and every rank reconstructs its coefficient block with
ctg_plan_crt_batch(curve_stride = Pb N, row_block = Pb, block_stride = B Pb N).  The
reassembled limbs must decode to exactly the one-shot resultants.  (Ranks run one after
another: no kernel waits on another rank's kernel, so one device is a faithful host.)
"""

import numpy as np
import pytest

import paper_1103_4697_b200 as P
from paper_1103_4697_b200 import curves, sharding

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G,kind,a,b", [(2, "dense", 12, 40), (3, "dense", 20, 64), (8, "dense", 16, 256),
                                       (8, "sheared", 2, 0)])
def test_sharded_pipeline_matches_one_shot(G, kind, a, b):
    import torch

    B = 5
    fs = [curves.make(kind, a, b, s) for s in range(1, B + 1)]
    pairs = [(f, curves.derive_y(f)) for f in fs]
    want = [P.resultant(*pq) for pq in pairs]
    plan = P.Plan(pairs)
    info = plan.info
    Pn, N, D, W = info["n_primes"], info["n_points"], info["n_coeffs"], info["out_limbs"] + 1
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    plan.upload(sh)
    Pb = sharding.prime_block(Pn, G, 0)[2]
    curve_stride, block_stride = sharding.strides(B, Pb, N)
    sends = []
    for r in range(G):
        k0, k1, _ = sharding.prime_block(Pn, G, r)
        send = torch.zeros((B, Pb, N), dtype=torch.int32, device="cuda")
        for s_ in (1, 2, 3):
            plan.stage(s_, k0, k1, send.data_ptr(), sh, curve_stride=Pb * N)
        sends.append(send)
    full = torch.stack(sends)  # the all-gather: [G][B][Pb][N]
    outs = []
    for r in range(G):
        j0, j1, Jb = sharding.coeff_block(D, G, r)
        out = torch.zeros((B * Jb * W,), dtype=torch.int32, device="cuda")
        if j1 > j0:
            plan.crt_batch(full.data_ptr(), j0, j1, out.data_ptr(), sh, curve_stride=curve_stride, row_block=Pb,
                           block_stride=block_stride)
        outs.append(out)
    torch.cuda.synchronize()
    plan.check(sh)
    gathered = np.stack([o.cpu().numpy().view("uint32") for o in outs])
    dense = sharding.reassemble(gathered, B, D, W, G)
    for bi in range(B):
        assert plan.decode(np.ascontiguousarray(dense[bi])) == want[bi], (G, kind, bi)


@pytest.mark.parametrize("G,mode", [(2, "fused"), (3, "fused"), (8, "fused"), (9, "fused"), (2, "copy"),
                                    (3, "copy")])
def test_c_abi_device_list_sharding(G, mode, monkeypatch):
    """The product path: ctg_resultant_batch with ctg_opts.n_devices = G (device 0 listed G
    times: the shards share the GPU).  Exchange "fused" (default, G <= 8): K4's epilogue stores
    each coefficient straight into the owning shard's receive block (peer stores across GPUs,
    local stores here); G = 9 and "copy": the all-gather of whole residue rows by device copies.
    Mixed shapes, a zero operand, a degree-0 operand and the d20/64 config (reference-pinned
    digest of seed 1) must equal the one-device call bit for bit."""
    import hashlib
    import json
    import os
    monkeypatch.setenv("CTG_SHARD_EXCHANGE", mode)
    pairs = []
    for s in range(1, 4):
        f = curves.make("dense", 12, 40, s)
        pairs.append((f, curves.derive_y(f)))
    f20 = curves.make("dense", 20, 64, 1)
    pairs.append((f20, curves.derive_y(f20)))
    fs = curves.make("sheared", 2, 0, 1)
    pairs.append((fs, curves.derive_y(fs)))
    pairs.append(({(1, 1): 3, (0, 0): -1}, {(2, 0): 1, (0, 2): 1, (0, 0): -4}))  # not a derivative pair
    pairs.append(({(0, 2): 1, (1, 0): -1}, {}))  # one zero operand -> zero polynomial
    pairs.append(({(0, 0): 5}, {(0, 3): 2, (1, 0): 1}))  # degree-0 operand
    want = P.resultant_batch(pairs)
    got = P.resultant_batch(pairs, devices=[0] * G)
    assert got == want
    gold = [json.loads(l) for l in open(os.path.join(os.path.dirname(__file__), "golden", "configs_big.jsonl"))]
    row = next(r for r in gold if r["curve"] == ["dense", 20, 64, 1])
    assert hashlib.sha256(",".join(format(c, "x") for c in got[3]).encode()).hexdigest() == row["sha256"]
    st = P.last_call_stats()
    assert st["kernel_launches"] > 0 and st["d2h_bytes"] > 0


def test_c_abi_comm_single_rank():
    """The multi-process path (ctg_opts.comm: libctg's own NCCL communicator, loaded at run time)
    with one rank: K4's by-destination send block, the grouped ncclSend / ncclRecv column swap
    and the all-gather of the CRT'd limb blocks are then copies to itself, and the result must
    equal the plain call (CTG_SHARD_EXCHANGE=nccl: the row all-gather instead).  (N ranks need
    N GPUs: NCCL refuses two ranks on one device.)"""
    pairs = []
    for s in range(1, 4):
        f = curves.make("dense", 12, 40, s)
        pairs.append((f, curves.derive_y(f)))
    pairs.append(({(0, 2): 1, (1, 0): -1}, {}))
    comm = P.Comm(1, 0, P.Comm.unique_id(), 0)
    try:
        assert P.resultant_batch(pairs, comm=comm) == P.resultant_batch(pairs)
    finally:
        comm.close()


@pytest.mark.parametrize("G,kind,a,b", [(2, "dense", 12, 40), (3, "dense", 20, 64), (8, "sheared", 2, 0)])
def test_sharded_column_exchange_matches_one_shot(G, kind, a, b):
    """The column-block exchange of the staged API (bench.py --gpus G): each rank's K4 writes by
    destination (ctg_plan_interp_cols: send = [G][B][Pb][Jb]), the all-to-all is emulated by
    taking block r of every rank's send for rank r, and ctg_plan_crt_cols reconstructs rank r's
    columns.  Reassembled, the limbs must decode to exactly the one-shot resultants."""
    import torch

    B = 4
    fs = [curves.make(kind, a, b, s) for s in range(1, B + 1)]
    pairs = [(f, curves.derive_y(f)) for f in fs]
    want = [P.resultant(*pq) for pq in pairs]
    plan = P.Plan(pairs)
    info = plan.info
    Pn, N, D, W = info["n_primes"], info["n_points"], info["n_coeffs"], info["out_limbs"] + 1
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    plan.upload(sh)
    Pb = sharding.prime_block(Pn, G, 0)[2]
    Jb = (D + G - 1) // G
    sends = []
    for r in range(G):
        k0, k1, _ = sharding.prime_block(Pn, G, r)
        rows = torch.zeros((B, Pb, N), dtype=torch.int32, device="cuda")
        send = torch.zeros((G, B, Pb, Jb), dtype=torch.int32, device="cuda")
        if k1 > k0:
            for s_ in (1, 2):
                plan.stage(s_, k0, k1, rows.data_ptr(), sh, curve_stride=Pb * N)
            plan.interp_cols(k0, k1, rows.data_ptr(), G, Pb, send.data_ptr(), sh, curve_stride=Pb * N)
        sends.append(send)
    outs = []
    for r in range(G):
        recv = torch.stack([sends[s_][r] for s_ in range(G)]).contiguous()  # the all-to-all
        j0, j1 = min(r * Jb, D), min((r + 1) * Jb, D)
        out = torch.zeros((B * max(j1 - j0, 1) * W,), dtype=torch.int32, device="cuda")
        if j1 > j0:
            plan.crt_cols(recv.data_ptr(), G, r, Pb, out.data_ptr(), sh)
        outs.append((j0, j1, out))
    torch.cuda.synchronize()
    plan.check(sh)
    dense = np.zeros((B, D, W), dtype=np.uint32)
    for j0, j1, out in outs:
        if j1 > j0:
            dense[:, j0:j1, :] = out.cpu().numpy().view("uint32").reshape(B, j1 - j0, W)
    for bi in range(B):
        assert plan.decode(np.ascontiguousarray(dense[bi])) == want[bi], (G, kind, bi)
