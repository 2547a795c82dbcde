"""Multi-GPU sharding of the hot path.

Two shardings, one process per GPU:

* **Independent block pairs** (the bench): every rank runs its own
  DiagABT/DiagATB pair; no collective on the data path (weak scaling).
* **Block-row data parallelism** (config 4, the 1024-row NAG step): rank r
  owns a contiguous range of the batch's 128-row block rows.  DiagABT,
  the softmax and the residual are local per block row; in DiagATB the
  ``row_sums`` block-row pre-add (encoding.py:375-377) is the only exchange:
  each rank pre-adds its own block rows, the per-rank pre-sums are summed
  over ranks as uint64 (R residues < 2^61 sum below 2^64) and reduced mod
  q_i.  Modular addition is associative, so the reduced ciphertext is
  residue-identical to a single-GPU pre-add over all block rows; everything
  after it (ladder, mask, conj, NAG update) is replicated and identical on
  every rank, so no broadcast is needed.

Encryption randomness: ranks draw nonces from disjoint ranges
(``rank_nonce_base``) so refreshes on different ranks never reuse a mask.
"""

from __future__ import annotations

import numpy as np

NONCE_STRIDE = 1 << 40


def rank_nonce_base(rank: int) -> int:
    return rank * NONCE_STRIDE


def partition(n_items: int, world: int, rank: int) -> range:
    """Contiguous near-even split of n_items (block rows) over ranks."""
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def mod_allreduce_host(residues: np.ndarray, moduli, group=None) -> np.ndarray:
    """Sum [2][l+1][N] uint64 residues over ranks (torch.distributed, any backend) and
    reduce limb i mod moduli[i].  Host-staged path (gloo / CPU tests)."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(residues).view(np.int64).copy())
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    out = t.numpy().view(np.uint64)
    q = np.asarray(moduli, dtype=np.uint64)[: out.shape[1]].reshape(1, -1, 1)
    return out % q


class _DeviceView:
    """__cuda_array_interface__ over a ciphertext's device residues (zero copy)."""

    def __init__(self, ptr: int, words: int):
        self.__cuda_array_interface__ = {"shape": (words,), "typestr": "<i8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class NcclModReducer:
    """Reducer for ``diag_atb(..., reducer=)`` / ``nag_step(..., reducer=)`` on GPUs:
    all-reduce (NCCL, SUM) of each pre-sum ciphertext's residues in place, then
    ``hc_mod_reduce`` on the library stream."""

    def __init__(self, group=None):
        self.group = group

    def __call__(self, ctx, handles):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _native as N

        L = N.lib()
        for h in handles:
            level = L.hc_ct_level(h)
            words = 2 * (level + 1) * ctx.N
            ptr = N.U64P()
            N.check(L.hc_ct_device_ptr(h, C.byref(ptr)))
            t = torch.as_tensor(_DeviceView(C.cast(ptr, C.c_void_p).value, words), device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        torch.cuda.current_stream().synchronize()
        for h in handles:
            N.check(L.hc_mod_reduce(ctx._h, h))


def local_rows(X: np.ndarray, grid_rows: int, world: int, rank: int) -> np.ndarray:
    """This rank's block rows of a batch (rows are padded to whole blocks by encode)."""
    n_blocks = -(-X.shape[0] // grid_rows)
    part = partition(n_blocks, world, rank)
    return X[part.start * grid_rows: min(X.shape[0], part.stop * grid_rows)]
