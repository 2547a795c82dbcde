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

Encryption randomness: ranks encrypt their own inputs with nonces from
disjoint ranges (``rank_nonce_base``).  Refreshes inside the sharded step
follow the whole batch's sequential nonce layout (``CKKSContext.set_shard``,
``hc_set_shard``), so the softmax refreshes of block row p draw the nonces a
single-context run of all block rows gives them, and the context nonce after
the softmax -- hence the replicated W / V refreshes -- is the same on every
rank: the weights stay bit-identical replicas without a broadcast.

Reducers: ``NcclModReducer`` (one process per GPU; collective and
``hc_mod_reduce`` ordered on the library stream, no host sync) and
``LocalModReducer`` (several shard contexts in one process, tests).
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


def check_sum_fits(world: int, moduli, level: int) -> None:
    """A sum of ``world`` canonical residues must fit a uint64 word (the
    all-reduce adds them as int64, wrapping like uint64)."""
    qmax = max(int(q) for q in list(moduli)[: level + 1])
    if world * qmax >= 1 << 64:
        raise ValueError(f"{world} ranks x {qmax.bit_length()}-bit primes overflow the uint64 sum")


def device_residues(ctx, handle):
    """int64 torch view of a ciphertext handle's [2][l+1][N] device residues."""
    import ctypes as C

    import torch

    from . import _native as N
    L = N.lib()
    level = L.hc_ct_level(handle)
    ptr = N.U64P()
    N.check(L.hc_ct_device_ptr(handle, C.byref(ptr)))
    words = 2 * (level + 1) * ctx.N
    return torch.as_tensor(_DeviceView(C.cast(ptr, C.c_void_p).value, words), device="cuda"), level


class NcclModReducer:
    """Reducer for ``diag_atb(..., reducer=)`` / ``nag_step(..., reducer=)`` on GPUs:
    an NCCL all-reduce (SUM) of each pre-sum ciphertext's residues in place,
    then ``hc_mod_reduce`` -- all ordered on the library's current stream
    (``hc_ctx_stream``): torch's NCCL stream waits for the pre-sums there and
    the stream waits for the collective, so the host never blocks and the
    next diagonal pass's work queues behind it."""

    def __init__(self, group=None):
        self.group = group

    def __call__(self, ctx, handles):
        import torch
        import torch.distributed as dist

        world = dist.get_world_size(self.group)
        stream = torch.cuda.ExternalStream(ctx.stream())
        with torch.cuda.stream(stream):
            for h in handles:
                t, level = device_residues(ctx, h)
                check_sum_fits(world, ctx.moduli, level)
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        for h in handles:
            ctx.mod_reduce(h)


class LocalModReducer:
    """The same exchange for ``world`` contexts driven from one process (one
    thread per shard, e.g. several shards on one GPU): each rank's pre-sums
    are summed as uint64 on the device, every rank receives the raw sum and
    finishes it with ``hc_mod_reduce`` (K8) -- the product's reduction kernel
    on genuinely unreduced words.  ``reducer.rank(r)`` is rank r's callable."""

    def __init__(self, world: int):
        import threading
        self.world = world
        self._bar = threading.Barrier(world)
        self._views = [None] * world
        self._sums = None

    def rank(self, r: int):
        return lambda ctx, handles: self._reduce(r, ctx, handles)

    def _reduce(self, r, ctx, handles):
        import torch
        ctx.sync()                                   # this rank's pre-sums are complete
        views = [device_residues(ctx, h) for h in handles]
        for _, level in views:
            check_sum_fits(self.world, ctx.moduli, level)
        self._views[r] = [v for v, _ in views]
        self._bar.wait()
        if r == 0:
            self._sums = [torch.stack([self._views[k][i] for k in range(self.world)]).sum(0)
                          for i in range(len(handles))]
            torch.cuda.synchronize()
        self._bar.wait()
        for v, s in zip(self._views[r], self._sums):
            v.copy_(s)
        torch.cuda.synchronize()
        self._bar.wait()                             # every rank has its copy
        for h in handles:
            ctx.mod_reduce(h)


def local_rows(X: np.ndarray, grid_rows: int, world: int, rank: int) -> np.ndarray:
    """This rank's block rows of a batch (rows are padded to whole blocks by encode)."""
    n_blocks = -(-X.shape[0] // grid_rows)
    part = partition(n_blocks, world, rank)
    return X[part.start * grid_rows: min(X.shape[0], part.stop * grid_rows)]
