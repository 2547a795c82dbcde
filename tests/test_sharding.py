"""Multi-process (gloo, world size 2) tests of the block-row sharding.

The DiagATB row_sums pre-add (encoding.py:375-377) is the only cross-rank
step; with the residues summed over ranks and reduced mod q_i, the sharded
product is residue-identical to the single-process one.  Runs the restated
reference schedule over the C RNS-CKKS oracle on CPU."""

import os
import socket

import numpy as np
import pytest

from paper_2403_14111_b200 import sharding


def test_partition_covers_all_rows():
    for n in (1, 7, 8, 9):
        for world in (1, 2, 3, 8):
            parts = [sharding.partition(n, world, r) for r in range(world)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(n))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    assert sharding.rank_nonce_base(1) - sharding.rank_nonce_base(0) == sharding.NONCE_STRIDE


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    rng = np.random.default_rng(5)
    A = rng.uniform(-1, 1, (64, 4))          # 4 block rows of 16, horizontally tiled (period 4)
    B = rng.uniform(-1, 1, (64, 21))         # 4 x 2 block grid
    return A, B


def _encode_all(ctx, A, B, S):
    ctx.nonce = 0
    EA = S.encode(ctx, A, "horizontal")
    EB = S.encode(ctx, B)
    return EA, EB


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    from oracle import rns as R
    from oracle import slots as S

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = R.OracleCKKSContext("small12", 16, seed=21)
    A, B = _inputs()
    EA, EB = _encode_all(ctx, A, B, S)
    rows = sharding.partition(EA.grid[0], world, rank)
    LA = S.Grid(ctx, EA.blocks[rows.start:rows.stop], EA.shape, EA.tiling, EA.period)
    LB = S.Grid(ctx, EB.blocks[rows.start:rows.stop], EB.shape, EB.tiling, EB.period)

    def presum(E, q):
        local = S.row_presum(E, q)
        red = sharding.mod_allreduce_host(local.data, ctx.p.moduli)
        return R.RnsBlock(ctx, red, local.level)

    out = S.diag_atb(LA, LB, scale=0.5, presum=presum)
    res = np.stack([b.data for b in out.blocks[0]])
    np.save(os.path.join(outdir, f"rank{rank}.npy"), res)
    dist.destroy_process_group()


def test_sharded_diag_atb_bit_exact_world2(tmp_path):
    import torch.multiprocessing as mp

    from oracle import rns as R
    from oracle import slots as S

    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    ctx = R.OracleCKKSContext("small12", 16, seed=21)
    A, B = _inputs()
    EA, EB = _encode_all(ctx, A, B, S)
    ref = S.diag_atb(EA, EB, scale=0.5)
    want = np.stack([b.data for b in ref.blocks[0]])
    r0 = np.load(tmp_path / "rank0.npy")
    r1 = np.load(tmp_path / "rank1.npy")
    np.testing.assert_array_equal(r0, want)
    np.testing.assert_array_equal(r1, want)
    vals = S.decode(ref, tol=1e-3)
    assert np.max(np.abs(vals - 0.5 * A.T @ B)) < 1e-3
