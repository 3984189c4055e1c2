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
