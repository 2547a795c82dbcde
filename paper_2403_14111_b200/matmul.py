"""DiagABT / DiagATB on the B200 backend (API of hefit.matmul, matmul.py:74-296).

Both products run as one native schedule call (csrc/schedules.cu) with the
reference's op order: ~350 primitive ops, each a handful of sm_100a kernels,
issued back to back on the context stream without returning to Python.
The executed ledger equals ``count_formula`` (Table 9 of the paper) exactly.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from .context import CKKSContext, Ciphertext, OP_KINDS
from .encoding import EncodedMatrix, next_pow2
from .errors import ShapeMismatch

ALGORITHMS = ("diag_abt", "diag_atb_rl", "diag_atb_pru", "col_major", "row_major", "jin_abt", "jin_atb")


def _lg(n):
    return int(math.log2(n))


def _native_ctx(*mats) -> CKKSContext:
    ctx = mats[0].ctx
    for M in mats:
        if M.ctx is not ctx:
            raise ShapeMismatch("operands from different contexts")
        if not isinstance(ctx, CKKSContext):
            raise TypeError("the B200 schedules need a CKKSContext")
        if not all(isinstance(b, Ciphertext) for row in M.blocks for b in row):
            raise TypeError("the B200 schedules take encrypted operands")
    return ctx


def _handles(blocks):
    arr = (C.c_void_p * len(blocks))()
    for i, b in enumerate(blocks):
        arr[i] = b._h
    return arr


def _apply_counts(ctx, counts):
    # the library already advanced the context counters; nothing to mirror
    return {k: int(counts[i]) for i, k in enumerate(OP_KINDS)}


def diag_abt(A: EncodedMatrix, B: EncodedMatrix, scale: float = 1.0) -> EncodedMatrix:
    """``scale * A B^T``: A (a x b) untiled, B (c x b) vertically tiled (matmul.py:74-110).

    Output (a x c) horizontally tiled with period c; consumes 3 levels."""
    if A.tiling != "none" or B.tiling != "vertical":
        raise ShapeMismatch(f"diag_abt: expected tilings (none, vertical), got ({A.tiling}, {B.tiling})")
    if A.shape[1] != B.shape[1]:
        raise ShapeMismatch(f"diag_abt: inner dims differ, {A.shape} vs {B.shape}")
    ctx = _native_ctx(A, B)
    c = B.period
    if c > ctx.grid_cols:
        raise ShapeMismatch(f"diag_abt: period {c} exceeds block columns {ctx.grid_cols}")
    m, n = A.grid
    if B.grid != (1, n):
        raise ShapeMismatch("diag_abt: B must be one block row matching A's block columns")
    out = (C.c_void_p * m)()
    counts = (C.c_int64 * N.NCOUNTS)()
    N.check(N.lib().hc_diag_abt(ctx._h, _handles(A.flat()), m, n, _handles(B.flat()), c, float(scale), out,
                                counts))
    blocks = tuple((Ciphertext(ctx, C.c_void_p(out[p])),) for p in range(m))
    return EncodedMatrix(ctx, blocks, (A.shape[0], B.shape[0]), "horizontal", c)


def diag_atb(A: EncodedMatrix, B: EncodedMatrix, scale: float = 1.0, reducer=None) -> EncodedMatrix:
    """``scale * A^T B``: A (a x c) horizontally tiled, B (a x b) untiled (matmul.py:113-154).

    RL branch when level(A) >= level(B), PRU otherwise.  ``reducer`` (multi-GPU)
    receives the block-row pre-sums (encoding.py:375-377) and must replace them
    by their modular sum over ranks (see ``sharding``)."""
    if A.tiling != "horizontal" or B.tiling != "none":
        raise ShapeMismatch(f"diag_atb: expected tilings (horizontal, none), got ({A.tiling}, {B.tiling})")
    if A.shape[0] != B.shape[0]:
        raise ShapeMismatch(f"diag_atb: outer dims differ, {A.shape} vs {B.shape}")
    ctx = _native_ctx(A, B)
    c = A.period
    if c > ctx.grid_rows or ctx.grid_rows % c:
        raise ShapeMismatch(f"diag_atb: period {c} incompatible with block rows {ctx.grid_rows}")
    m, n = B.grid
    if A.grid != (m, 1):
        raise ShapeMismatch("diag_atb: A must be one block column matching B's block rows")
    out = (C.c_void_p * n)()
    counts = (C.c_int64 * N.NCOUNTS)()
    cb = N.REDUCE_FN(0) if reducer is None else _reduce_callback(ctx, reducer)
    N.check(N.lib().hc_diag_atb(ctx._h, _handles(A.flat()), m, _handles(B.flat()), n, c, float(scale), out,
                                counts, cb, None))
    blocks = (tuple(Ciphertext(ctx, C.c_void_p(out[q])) for q in range(n)),)
    return EncodedMatrix(ctx, blocks, (A.shape[1], B.shape[1]), "vertical", c)


def col_major_abt(A: EncodedMatrix, B: EncodedMatrix, scale: float = 1.0) -> EncodedMatrix:
    """Table-4 baseline ``scale * A B^T`` with both operands untiled (matmul.py:160-198):
    one mask-replicate-reduce pass per row of B; 3 levels."""
    if A.tiling != "none" or B.tiling != "none":
        raise ShapeMismatch("col_major_abt: expected untiled operands")
    if A.shape[1] != B.shape[1]:
        raise ShapeMismatch(f"col_major_abt: inner dims differ, {A.shape} vs {B.shape}")
    ctx = _native_ctx(A, B)
    c = B.shape[0]
    m, n = A.grid
    if B.grid != (1, n) or c > ctx.grid_cols:
        raise ShapeMismatch(f"col_major_abt: B rows {c} must fit one block and {ctx.grid_cols} columns")
    out = (C.c_void_p * m)()
    counts = (C.c_int64 * N.NCOUNTS)()
    N.check(N.lib().hc_col_major_abt(ctx._h, _handles(A.flat()), m, n, _handles(B.flat()), c, float(scale), out,
                                     counts))
    blocks = tuple((Ciphertext(ctx, C.c_void_p(out[p])),) for p in range(m))
    return EncodedMatrix(ctx, blocks, (A.shape[0], c), "none", None)


def row_major_atb(A: EncodedMatrix, B: EncodedMatrix, scale: float = 1.0) -> EncodedMatrix:
    """Table-4 baseline ``scale * A^T B`` with both operands untiled (matmul.py:201-237):
    one pass per column of A; 3 levels."""
    if A.tiling != "none" or B.tiling != "none":
        raise ShapeMismatch("row_major_atb: expected untiled operands")
    if A.shape[0] != B.shape[0]:
        raise ShapeMismatch(f"row_major_atb: outer dims differ, {A.shape} vs {B.shape}")
    ctx = _native_ctx(A, B)
    c = A.shape[1]
    m, n = B.grid
    if A.grid != (m, 1) or c > ctx.grid_rows:
        raise ShapeMismatch(f"row_major_atb: A columns {c} must fit one block and {ctx.grid_rows} rows")
    out = (C.c_void_p * n)()
    counts = (C.c_int64 * N.NCOUNTS)()
    N.check(N.lib().hc_row_major_atb(ctx._h, _handles(A.flat()), m, _handles(B.flat()), n, c, float(scale), out,
                                     counts))
    blocks = (tuple(Ciphertext(ctx, C.c_void_p(out[q])) for q in range(n)),)
    return EncodedMatrix(ctx, blocks, (c, B.shape[1]), "none", None)


def _reduce_callback(ctx, reducer):
    def cb(_user, cts, count):
        try:
            hs = [cts[i] for i in range(count)]
            reducer(ctx, hs)
            return 0
        except Exception:  # surfaced as HC_ECUDA by the library
            import traceback
            traceback.print_exc()
            return -1
    fn = N.REDUCE_FN(cb)
    _reduce_callback._keep = fn      # keep the thunk alive for the call
    return fn


def count_formula(algorithm: str, shape, s0: int, s1: int):
    """Closed-form {CMult, Mult, Rot} (matmul.py:253-296, paper Table 9)."""
    a, b, c = (int(v) for v in shape)
    if min(a, b, c) < 1:
        raise ShapeMismatch(f"count_formula: bad shape {shape}")
    m, n = -(-a // s0), -(-b // s1)
    l0, l1, h = _lg(s0), _lg(s1), c // 2
    if algorithm == "diag_abt":
        if c == 1:
            return {"CMult": 2 * m, "Mult": m * n, "Rot": 2 * m * l1}
        return {"CMult": c * m, "Mult": h * m * n, "Rot": h * (n + 2 * m * l1)}
    if algorithm == "diag_atb_rl":
        if c == 1:
            return {"CMult": n, "Mult": m * n, "Rot": n * l0}
        return {"CMult": h * (m + n), "Mult": h * m * n, "Rot": h * (2 * m + n * l0)}
    if algorithm == "diag_atb_pru":
        if c == 1:
            return {"CMult": n, "Mult": m * n, "Rot": n * l0}
        return {"CMult": m + (h - 1) * m * n + h * n, "Mult": h * m * n,
                "Rot": 2 * m + (h - 1) * (m + m * n) + h * n * l0}
    if algorithm in ("col_major", "row_major"):
        return {"CMult": c * (n + m), "Mult": c * m * n, "Rot": c * (n * l0 + m * l1 + m) - m}
    if algorithm == "jin_abt":
        return {"CMult": 0, "Mult": b * c, "Rot": 0}
    if algorithm == "jin_atb":
        return {"CMult": 0, "Mult": b * c, "Rot": b * c * _lg(s0 * s1)}
    raise ShapeMismatch(f"count_formula: unknown algorithm {algorithm!r}")


def expected_period(c: int) -> int:
    return next_pow2(c)


def ladder_amounts(ctx, stride: int, steps: int):
    """Rotation amounts of the doubling ladder (stride, steps): with the fused
    schedule forms (``ctx.hoist``) the rotate-and-sum stages' u * s, u < 2^w
    (w = 3, 2 or 1 steps per stage, s = stride * 2^t), else stride * 2^t."""
    S = ctx.slot_count
    if not getattr(ctx, "hoist", False):
        return {(stride * (1 << t)) % S for t in range(steps)}
    out, t = set(), 0
    while t < steps:
        rem = steps - t
        w = 3 if (rem >= 5 or rem == 3) else min(2, rem)
        out |= {(stride * (1 << t) * u) % S for u in range(1, 1 << w)}
        t += w
    return out


def rotation_steps(ctx, algorithm: str, c: int, m: int = 1, n: int = 1):
    """Left-rotation amounts a schedule will use (to pre-generate keys)."""
    s0, s1, S = ctx.grid_rows, ctx.grid_cols, ctx.slot_count
    steps = set()
    if algorithm == "diag_abt":
        steps |= ladder_amounts(ctx, 1, _lg(s1)) | ladder_amounts(ctx, -1, _lg(s1))
        for k in range(1, c // 2 + 1):
            steps.add((k % s0) * s1)
    else:
        steps |= ladder_amounts(ctx, s1, _lg(s0))
        steps |= {S - s1, s1}
        for k in range(1, c // 2 + 1):
            steps.add(k % s1)
    steps.discard(0)
    return sorted(steps)
