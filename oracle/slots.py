"""TEST INFRASTRUCTURE ONLY — slot-level restatement of the reference algorithm.

This module is part of the parity oracle.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import
it; the product package never does.

It restates, in plain numpy, the reference ``hefit`` package's hot path
(``/root/reference/pkg/src/hefit``) with the same operation order:

* L0 ``SlotBackend`` — the float64 slot emulator (``emulator.py:111-281``):
  level rules, auto-bootstrap per operand (``emulator.py:184-191``), the op
  ledger (``emulator.py:70-108``).
* L1 ``Grid`` + ``encode``/``decode``/masks/``rot_up``/``rot_left``/
  ``prot_up``/``col_sums``/``row_sums`` (``encoding.py:38-381``).
* L2 ``diag_abt``/``diag_atb``/``count_formula`` (``matmul.py:74-154,253-296``)
  and the approximate softmax (``approx.py:195-344``).
* L3 ``nag_step`` (``training.py:66-100``) and the float64 twin
  (``plainref.py:21-96``).

Every schedule function takes any context object implementing the
``EmulatorContext`` duck type, so the same restated schedule can be driven
over (a) ``SlotBackend`` — pinned bit-for-bit against golden vectors produced
by the reference itself (``tests/golden/make_golden.py``), (b) the C RNS-CKKS
oracle (``oracle/rns.py``), or (c) the product's CUDA ``CKKSContext`` (the
drop-in test: the reference's op sequence issued op by op through the
product's backend interface).
"""

from __future__ import annotations

import math
import threading

import numpy as np

OP_KINDS = ("Add", "CMult", "Mult", "Rot", "Conj", "Bootstrap")
WEIGHTS_MS = {"Add": 0.085, "CMult": 0.9, "Mult": 1.6, "Rot": 1.2, "Conj": 1.2,
              "Bootstrap": 159.0}                                   # emulator.py:33-40
PLAIN_LEVEL = math.inf
IMAG_TOL = 1e-9                                                     # encoding.py:25


class OracleError(Exception):
    code = "oracle"


class DepthExhausted(OracleError):
    code = "emulator.depth"


class SlotCountMismatch(OracleError):
    code = "emulator.slots"


class ShapeMismatch(OracleError):
    code = "encoding.shape"


class TilingError(OracleError):
    code = "encoding.tiling"


class ResidualImaginary(OracleError):
    code = "encoding.imaginary"


def npow2(n: int) -> int:
    return 1 << (int(n) - 1).bit_length()


def lg(n: int) -> int:
    return int(math.log2(n))


# ---------------------------------------------------------------------------
# L0: ledger + float64 slot backend
# ---------------------------------------------------------------------------


class Ledger:
    def __init__(self):
        self.c = dict.fromkeys(OP_KINDS, 0)
        self._lock = threading.Lock()

    def record(self, kind, n=1):
        with self._lock:
            self.c[kind] += n

    def counts(self):
        with self._lock:
            return dict(self.c)

    snapshot = counts

    def delta(self, before):
        now = self.counts()
        return {k: now[k] - before.get(k, 0) for k in OP_KINDS}

    def reset(self):
        with self._lock:
            for k in OP_KINDS:
                self.c[k] = 0

    @property
    def estimated_ms(self):
        return float(sum(v * WEIGHTS_MS[k] for k, v in self.counts().items()))


class Slots:
    """emulator.py:49-67 — an immutable slot vector with a level."""

    __slots__ = ("slots", "level", "encrypted")

    def __init__(self, slots, level, encrypted=True):
        a = np.ascontiguousarray(np.asarray(slots, dtype=np.complex128))
        a.setflags(write=False)
        self.slots, self.level, self.encrypted = a, level, encrypted

    def __len__(self):
        return self.slots.shape[0]


class SlotBackend:
    """Restates EmulatorContext (emulator.py:111-281) op for op."""

    def __init__(self, slot_count=4096, grid_rows=64, *, max_level=12, auto_bootstrap=False):
        self.slot_count = slot_count
        self.grid_rows = grid_rows
        self.grid_cols = slot_count // grid_rows
        self.max_level = max_level
        self.auto_bootstrap = auto_bootstrap
        self.ledger = Ledger()
        self.decode_events = []

    def _vec(self, v):
        a = np.asarray(v, dtype=np.complex128).ravel()
        if a.shape[0] != self.slot_count:
            raise SlotCountMismatch(f"expected {self.slot_count} slots, got {a.shape[0]}")
        return a

    def encrypt(self, values, level=None):
        lv = self.max_level if level is None else level
        if not 0 <= lv <= self.max_level:
            raise ValueError(f"level must be in [0, {self.max_level}], got {lv}")
        return Slots(self._vec(values), lv, True)

    def pack(self, values):
        return Slots(self._vec(values), PLAIN_LEVEL, False)

    def _op(self, v):                                               # emulator.py:172-182
        if isinstance(v, Slots):
            if len(v) != self.slot_count:
                raise SlotCountMismatch("width")
            return v.slots, v.encrypted, v.level
        if isinstance(v, (int, float, complex, np.integer, np.floating, np.complexfloating)):
            return complex(v), False, PLAIN_LEVEL
        return self._vec(v), False, PLAIN_LEVEL

    def _ready(self, lv, enc, op):                                  # emulator.py:184-191
        if not enc or lv >= 1:
            return lv
        if self.auto_bootstrap:
            self.ledger.record("Bootstrap")
            return self.max_level
        raise DepthExhausted(f"{op}: operand at level {int(lv)}")

    def add(self, x, y):
        vx, ex, lx = self._op(x)
        vy, ey, ly = self._op(y)
        if ex or ey:
            self.ledger.record("Add")
        return Slots(vx + vy, min(lx, ly), ex or ey)

    def sub(self, x, y):
        vx, ex, lx = self._op(x)
        vy, ey, ly = self._op(y)
        if ex or ey:
            self.ledger.record("Add")
        return Slots(vx - vy, min(lx, ly), ex or ey)

    def mult(self, x, y):
        vx, ex, lx = self._op(x)
        vy, ey, ly = self._op(y)
        if ex:
            lx = self._ready(lx, ex, "mult")
        if ey:
            ly = self._ready(ly, ey, "mult")
        if ex and ey:
            self.ledger.record("Mult")
        elif ex or ey:
            self.ledger.record("CMult")
        lv = min(lx, ly) - (1 if (ex or ey) else 0)
        return Slots(vx * vy, lv, ex or ey)

    def cmult(self, x, y):
        if isinstance(y, Slots) and y.encrypted:
            raise TypeError("cmult expects a plaintext second operand")
        return self.mult(x, y)

    def lrot(self, x, r):
        vx, ex, lx = self._op(x)
        r = int(r) % self.slot_count
        if r == 0:
            return x if isinstance(x, Slots) else Slots(vx, lx, ex)
        if ex:
            self.ledger.record("Rot")
        return Slots(np.roll(vx, -r), lx, ex)

    def rrot(self, x, r):
        return self.lrot(x, -int(r))

    def conj(self, x):
        vx, ex, lx = self._op(x)
        if ex:
            self.ledger.record("Conj")
        return Slots(np.conj(vx), lx, ex)

    def mul_i(self, x):
        vx, ex, lx = self._op(x)
        return Slots(vx * 1j, lx, ex)

    def bootstrap(self, x):
        if not isinstance(x, Slots) or not x.encrypted:
            return x
        self.ledger.record("Bootstrap")
        return Slots(x.slots, self.max_level, True)

    def note_decode(self, role, tag=None):
        self.decode_events.append((role, tag))

    def decodes_by(self, role):
        return [e for e in self.decode_events if e[0] == role]


# ---------------------------------------------------------------------------
# L1: block grids (encoding.py)
# ---------------------------------------------------------------------------


class Grid:
    """encoding.py:38-132 — block grid plus logical shape and tiling."""

    def __init__(self, ctx, blocks, shape, tiling="none", period=None):
        self.ctx = ctx
        self.blocks = tuple(tuple(r) for r in blocks)
        self.shape = tuple(int(s) for s in shape)
        self.tiling, self.period = tiling, period

    @property
    def grid(self):
        return len(self.blocks), len(self.blocks[0])

    @property
    def encrypted(self):
        return self.blocks[0][0].encrypted

    @property
    def level(self):
        return min(b.level for r in self.blocks for b in r)

    def meta(self, shape=None, tiling=None, period=None):
        return Grid(self.ctx, self.blocks, self.shape if shape is None else shape,
                    self.tiling if tiling is None else tiling,
                    self.period if period is None else period)

    def each(self, fn):
        return Grid(self.ctx, [[fn(b) for b in r] for r in self.blocks], self.shape,
                    self.tiling, self.period)

    def zip(self, other, fn):
        if isinstance(other, Grid):
            if other.grid != self.grid:
                raise ShapeMismatch("grid")
            nb = [[fn(a, b) for a, b in zip(ra, rb)] for ra, rb in zip(self.blocks, other.blocks)]
        else:
            nb = [[fn(a, other) for a in r] for r in self.blocks]
        return Grid(self.ctx, nb, self.shape, self.tiling, self.period)

    def add(self, o):
        return self.zip(o, self.ctx.add)

    def sub(self, o):
        return self.zip(o, self.ctx.sub)

    def rsub(self, o):
        return self.zip(o, lambda a, b: self.ctx.sub(b, a))

    def mul(self, o):
        return self.zip(o, self.ctx.mult)

    def scale(self, t):
        return self.each(lambda b: self.ctx.cmult(b, t))

    def lrot(self, r):
        return self.each(lambda b: self.ctx.lrot(b, r))

    def rrot(self, r):
        return self.each(lambda b: self.ctx.rrot(b, r))

    def conj(self):
        return self.each(self.ctx.conj)

    def bootstrap(self):
        return self.each(self.ctx.bootstrap)


def layout(ctx, values, tiling="none"):
    """encoding.py:138-192 — the padded/tiled float64 grid and its block split."""
    arr = np.asarray(values, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ShapeMismatch(f"bad shape {arr.shape}")
    rows, cols = arr.shape
    s0, s1 = ctx.grid_rows, ctx.grid_cols
    period = None
    if tiling == "vertical":
        period = npow2(rows)
        if period > s0:
            raise TilingError("rows")
        t = np.zeros((period, cols))
        t[:rows] = arr
        arr, rows = np.tile(t, (s0 // period, 1)), s0
    elif tiling == "horizontal":
        period = npow2(cols)
        if period > s1:
            raise TilingError("cols")
        t = np.zeros((rows, period))
        t[:, :cols] = arr
        arr, cols = np.tile(t, (1, s1 // period)), s1
    elif tiling != "none":
        raise TilingError(tiling)
    gr, gc = -(-rows // s0), -(-cols // s1)
    pad = np.zeros((gr * s0, gc * s1))
    pad[:rows, :cols] = arr
    parts = [[pad[p * s0:(p + 1) * s0, q * s1:(q + 1) * s1].ravel() for q in range(gc)]
             for p in range(gr)]
    return parts, period


def encode(ctx, values, tiling="none", encrypted=True, level=None):
    parts, period = layout(ctx, values, tiling)
    mk = (lambda v: ctx.encrypt(v, level)) if encrypted else ctx.pack
    shp = np.asarray(values).shape
    return Grid(ctx, [[mk(v) for v in r] for r in parts], shp, tiling, period)


def grid_slots(G, slot_reader=None):
    """encoding.py:196-205 — padded complex grid (slot_reader decrypts a block)."""
    ctx = G.ctx
    s0, s1 = ctx.grid_rows, ctx.grid_cols
    gr, gc = G.grid
    out = np.empty((gr * s0, gc * s1), dtype=np.complex128)
    for p in range(gr):
        for q in range(gc):
            b = G.blocks[p][q]
            v = slot_reader(b) if slot_reader is not None else b.slots
            out[p * s0:(p + 1) * s0, q * s1:(q + 1) * s1] = np.asarray(v).reshape(s0, s1)
    return out


def decode(G, role="observer", tag=None, tol=IMAG_TOL, slot_reader=None):
    if G.encrypted:
        G.ctx.note_decode(role, tag)
    full = grid_slots(G, slot_reader)
    lo = full[:G.shape[0], :G.shape[1]]
    worst = float(np.max(np.abs(lo.imag))) if lo.size else 0.0
    if worst >= tol:
        raise ResidualImaginary(f"imag residue {worst:.3e}")
    return np.array(lo.real, dtype=np.float64)


def pattern(ctx, pat, grid=(1, 1)):
    pat = np.asarray(pat)
    if pat.shape != (ctx.grid_rows, ctx.grid_cols):
        raise ShapeMismatch("pattern")
    blk = ctx.pack(pat.ravel())
    gr, gc = grid
    return Grid(ctx, [[blk] * gc for _ in range(gr)], (gr * ctx.grid_rows, gc * ctx.grid_cols))


def diag_pattern(s0, s1, shift, modulus, complexified=False, scale=1.0):
    """encoding.py:244-271 as a bare array."""
    shift = int(shift) % modulus
    i = np.arange(s0)[:, None]
    j = np.arange(s1)[None, :]
    main = ((j - i - shift) % modulus == 0).astype(np.complex128)
    if complexified:
        twin = ((j - i - shift - modulus // 2) % modulus == 0).astype(np.complex128)
        pat = 0.5 * main - 0.5j * twin
    else:
        pat = main
    return pat * scale


def make_mask(ctx, shift, modulus, grid=(1, 1), complexified=False, scale=1.0):
    s0, s1 = ctx.grid_rows, ctx.grid_cols
    if modulus < 1 or s0 % modulus or s1 % modulus:
        raise ShapeMismatch("mask modulus")
    return pattern(ctx, diag_pattern(s0, s1, shift, modulus, complexified, scale), grid)


def keep_head_pattern(s0, s1, stop, start=0):
    """encoding.py:274-278 — columns start <= j < stop."""
    j = np.arange(s1)
    return np.broadcast_to(np.where((j >= start) & (j < stop), 1.0, 0.0), (s0, s1))


def rot_up(E, k):                                                   # encoding.py:284-289
    k = int(k) % E.ctx.grid_rows
    return E if k == 0 else E.lrot(k * E.ctx.grid_cols)


def rot_left(E, k, first=None):                                     # encoding.py:291-311
    """``first(b)`` (default ``lrot(b, k)``) supplies the leading rotation,
    so a caller can hoist it across several k (fused form, ``diag_atb``)."""
    ctx, s1 = E.ctx, E.ctx.grid_cols
    k = int(k) % s1
    if k == 0:
        return E
    keep = ctx.pack(keep_head_pattern(ctx.grid_rows, s1, s1 - k).ravel())

    def fix(b):
        a1 = ctx.lrot(b, k) if first is None else first(b)
        head = ctx.cmult(a1, keep)
        tail = ctx.sub(a1, head)
        return ctx.add(head, ctx.rrot(tail, s1))
    return E.each(fix)


def prot_up(E, k):                                                  # encoding.py:314-332
    ctx, s1 = E.ctx, E.ctx.grid_cols
    k = int(k) % s1
    if k == 0:
        return E
    keep = ctx.pack(keep_head_pattern(ctx.grid_rows, s1, s1 - k).ravel())

    def fix(b):
        head = ctx.cmult(b, keep)
        tail = ctx.sub(b, head)
        return ctx.add(head, ctx.lrot(tail, s1))
    return E.each(fix)


def ladder_plan(steps):
    """Doubling steps per rotate-and-sum stage: radix 8 (3 steps, 7 rotations)
    while at least 5 steps remain or exactly 3, else radix 4 (2 steps), else a
    single step -- 8 -> 3 + 3 + 2, 7 -> 3 + 2 + 2.  A stage costs one ModUp +
    ModDown plus a key product per rotation (~1/9 of the pair each at cfg1),
    so a third step per stage pays for its four extra key products, a lone
    trailing step never does."""
    plan, rem = [], steps
    while rem > 0:
        w = 3 if (rem >= 5 or rem == 3) else min(2, rem)
        plan.append(w)
        rem -= w
    return plan


def ladder(ctx, acc, stride, steps):
    """The reference's doubling ladder ``for t < steps: acc = add(acc,
    lrot(acc, stride * 2^t))`` (stride < 0: rrot) -- encoding.py:354-359,
    378-379, approx.py:165-189.  On a context with the fused schedule forms
     w = 2 or 3 steps (``ladder_plan``) become one rotate-and-sum
    stage ``acc + sum_{u < 2^w} lrot(acc, u s)``, s = stride * 2^t: the same
    slot values and ledger, one ModUp / ModDown per stage."""
    if getattr(ctx, "hoist", False) and hasattr(ctx, "ladder") and ctx._kind(acc)[0] == "ct":
        return ctx.ladder(acc, stride, steps)       # the CUDA product's own ladder (same stages)
    if getattr(ctx, "hoist", False) and hasattr(ctx, "rotsum") and ctx._kind(acc)[0] == "ct":
        t = 0
        for w in ladder_plan(steps):
            base = stride * (1 << t)
            acc = ctx.rotsum(acc, [base * u for u in range(1, 1 << w)], w)
            t += w
        return acc
    for t in range(steps):
        acc = ctx.add(acc, ctx.lrot(acc, stride * (1 << t)))
    return acc


def col_ladder(ctx, acc):
    """encoding.py:354-359 — lrot ladder, column-0 mask, rrot ladder."""
    s1 = ctx.grid_cols
    c0 = np.zeros((ctx.grid_rows, s1))
    c0[:, 0] = 1.0
    c0b = ctx.pack(c0.ravel())
    acc = ladder(ctx, acc, 1, lg(s1))
    acc = ctx.cmult(acc, c0b)
    acc = ladder(ctx, acc, -1, lg(s1))
    return acc


def col_sums(E):                                                    # encoding.py:335-360
    ctx = E.ctx
    gr, gc = E.grid
    rows = []
    for p in range(gr):
        acc = E.blocks[p][0]
        for q in range(1, gc):
            acc = ctx.add(acc, E.blocks[p][q])
        rows.append((col_ladder(ctx, acc),))
    return Grid(ctx, rows, (E.shape[0], ctx.grid_cols))


def row_presum(E, q):
    """encoding.py:375-377 — the block-row pre-add (cross-rank reduction point)."""
    ctx = E.ctx
    acc = E.blocks[0][q]
    for p in range(1, E.grid[0]):
        acc = ctx.add(acc, E.blocks[p][q])
    return acc


def row_ladder(ctx, acc):
    """encoding.py:378-379 — log2(s0) row-rotation doubling ladder."""
    return ladder(ctx, acc, ctx.grid_cols, lg(ctx.grid_rows))


def row_sums(E, presum=row_presum):                                 # encoding.py:363-381
    ctx = E.ctx
    cols = [row_ladder(ctx, presum(E, q)) for q in range(E.grid[1])]
    return Grid(ctx, (tuple(cols),), (ctx.grid_rows, E.shape[1]))


# ---------------------------------------------------------------------------
# L2: products (matmul.py)
# ---------------------------------------------------------------------------


def _rowwise(A, R):
    ctx = A.ctx
    return Grid(ctx, [[ctx.mult(A.blocks[p][q], R.blocks[0][q]) for q in range(A.grid[1])]
                      for p in range(A.grid[0])], A.shape)


def _colwise(C, B):
    ctx = B.ctx
    return Grid(ctx, [[ctx.mult(C.blocks[p][0], B.blocks[p][q]) for q in range(B.grid[1])]
                      for p in range(B.grid[0])], B.shape)


def fused(ctx, depth, *grids):
    """Whether the fused schedule forms apply: the context
    offers them (the RNS oracle or the CUDA product with ``hoist`` on) and no
    auto-bootstrap can fire inside the product, which consumes ``depth - 1``
    levels — the CUDA product's lockstep condition (csrc/schedules.cu)."""
    return (getattr(ctx, "hoist", False) and hasattr(ctx, "lrot_hoisted")
            and (not ctx.auto_bootstrap or min(g.level for g in grids) >= depth))


def diag_abt(A, B, scale=1.0):                                      # matmul.py:74-110
    if A.tiling != "none" or B.tiling != "vertical" or A.shape[1] != B.shape[1]:
        raise ShapeMismatch("diag_abt layout")
    ctx, c, m = A.ctx, B.period, A.grid[0]
    out_shape = (A.shape[0], B.shape[0])
    if c == 1:
        sums = col_sums(_rowwise(A, B))
        return sums.mul(make_mask(ctx, 0, 1, (m, 1), scale=scale)).meta(out_shape, "horizontal", 1)
    rolled = rot_up(B, c // 2)
    packed = B.add(rolled.each(ctx.mul_i))
    acc = None
    if fused(ctx, 4, A, B) and packed.grid[0] == 1:
        # fused form: the c/2 rotations RU(packed, k) of a block column share
        # one ModUp, and each block row's product sum (the col_sums pre-add of
        # the rowwise products) is relinearised and rescaled once
        s0, s1, n = ctx.grid_rows, ctx.grid_cols, packed.grid[1]
        rots = [ctx.lrot_hoisted(packed.blocks[0][q], [(k % s0) * s1 for k in range(c // 2)]) for q in range(n)]
        for k in range(c // 2):
            rows = [(col_ladder(ctx, ctx.mult_sum(list(A.blocks[p]), [rots[q][k] for q in range(n)])),)
                    for p in range(m)]
            sums = Grid(ctx, rows, (A.shape[0], s1))
            term = sums.mul(make_mask(ctx, k, c, (m, 1), True, scale))
            acc = term if acc is None else acc.add(term)
        return acc.add(acc.conj()).meta(out_shape, "horizontal", c)
    for k in range(c // 2):
        sums = col_sums(_rowwise(A, rot_up(packed, k)))
        term = sums.mul(make_mask(ctx, k, c, (m, 1), True, scale))
        acc = term if acc is None else acc.add(term)
    return acc.add(acc.conj()).meta(out_shape, "horizontal", c)


def diag_atb(A, B, scale=1.0, presum=row_presum):                   # matmul.py:113-154
    if A.tiling != "horizontal" or B.tiling != "none" or A.shape[0] != B.shape[0]:
        raise ShapeMismatch("diag_atb layout")
    ctx, c, n = A.ctx, A.period, B.grid[1]
    out_shape = (A.shape[1], B.shape[1])
    if c == 1:
        sums = row_sums(_colwise(A, B), presum)
        return sums.mul(make_mask(ctx, 0, 1, (1, n), scale=scale)).meta(out_shape, "vertical", 1)
    partial = A.level < B.level
    packed = A.add(rot_left(A, c // 2).each(ctx.mul_i))
    acc = None
    hoisted = None
    if fused(ctx, 5, A, B):
        # fused form: the per-pass leading rotations lrot(packed, k) of a block
        # share one ModUp
        s1 = ctx.grid_cols
        amounts = [k if partial else k % s1 for k in range(c // 2)]
        hoisted = {id(b): ctx.lrot_hoisted(b, amounts) for r in packed.blocks for b in r}
    for k in range(c // 2):
        if hoisted is not None:
            pick = (lambda kk: (lambda b: hoisted[id(b)][kk]))(k)
            if partial:
                left, right = packed.each(pick), prot_up(B, k)
            else:
                left, right = rot_left(packed, k, first=pick), B
        elif partial:
            left, right = packed.lrot(k), prot_up(B, k)
        else:
            left, right = rot_left(packed, k), B
        sums = row_sums(_colwise(left, right), presum)
        term = sums.mul(make_mask(ctx, -k, c, (1, n), True, scale))
        acc = term if acc is None else acc.add(term)
    return acc.add(acc.conj()).meta(out_shape, "vertical", c)


def col_major_abt(A, B, scale=1.0):                                 # matmul.py:160-198
    """Table-4 baseline: one mask-replicate-reduce pass per row j of B."""
    if A.tiling != "none" or B.tiling != "none" or A.shape[1] != B.shape[1]:
        raise ShapeMismatch("col_major_abt layout")
    ctx = A.ctx
    s0, s1 = ctx.grid_rows, ctx.grid_cols
    c = B.shape[0]
    if B.grid[0] != 1 or c > s1:
        raise ShapeMismatch("col_major_abt: B must fit one block row")
    m, n = A.grid
    c0 = np.zeros((s0, s1))
    c0[:, 0] = scale
    c0b = ctx.pack(c0.ravel())
    acc = None
    for j in range(c):
        rowj = np.zeros((s0, s1))
        rowj[j, :] = 1.0
        picked = B.mul(pattern(ctx, rowj, B.grid))
        picked = picked.each(lambda b: ladder(ctx, b, s1, lg(s0)))
        prod = _rowwise(A, picked)
        folded = []
        for p in range(m):
            blk = prod.blocks[p][0]
            for q in range(1, n):
                blk = ctx.add(blk, prod.blocks[p][q])
            blk = ladder(ctx, blk, 1, lg(s1))
            blk = ctx.cmult(blk, c0b)
            blk = ctx.rrot(blk, j)
            folded.append((blk,))
        term = Grid(ctx, folded, (A.shape[0], c))
        acc = term if acc is None else acc.add(term)
    return acc.meta((A.shape[0], c))


def row_major_atb(A, B, scale=1.0):                                 # matmul.py:201-237
    """Table-4 baseline: one pass per column j of A."""
    if A.tiling != "none" or B.tiling != "none" or A.shape[0] != B.shape[0]:
        raise ShapeMismatch("row_major_atb layout")
    ctx = A.ctx
    s0, s1 = ctx.grid_rows, ctx.grid_cols
    c = A.shape[1]
    if A.grid[1] != 1 or c > s0:
        raise ShapeMismatch("row_major_atb: A must fit one block column")
    n = B.grid[1]
    c0 = np.zeros((s0, s1))
    c0[:, 0] = 1.0
    c0b = ctx.pack(c0.ravel())
    acc = None
    for j in range(c):
        picked = A.lrot(j)
        picked = picked.each(lambda b: ctx.cmult(b, c0b))
        picked = picked.each(lambda b: ladder(ctx, b, -1, lg(s1)))
        sums = row_sums(_colwise(picked, B))
        rowj = np.zeros((s0, s1))
        rowj[j, :] = scale
        term = sums.mul(pattern(ctx, rowj, (1, n)))
        acc = term if acc is None else acc.add(term)
    return acc.meta((c, B.shape[1]))


def count_formula(algorithm, shape, s0, s1):                        # matmul.py:253-296
    a, b, c = (int(v) for v in shape)
    m, n = -(-a // s0), -(-b // s1)
    l0, l1, h = lg(s0), lg(s1), c // 2
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
    raise ShapeMismatch(algorithm)


# ---------------------------------------------------------------------------
# L2: softmax (approx.py), encrypted carrier and float64 array carrier
# ---------------------------------------------------------------------------

EXP_POLY = (                                                        # _constants.py:7-21
    0.9999999999999948, 0.9999999999996788, 0.5000000000004744, 0.1666666666766445,
    0.04166666666019774, 0.00833333324592319, 0.0013888889188354027,
    0.00019841302319140728, 2.4801530417934142e-05, 2.7551504280360845e-06,
    2.7561173628426655e-07, 2.5547752396936175e-08, 2.0934824859870782e-09,
)
COMP_F = (35 / 16, -35 / 16, 21 / 16, -5 / 16)                     # approx.py:34-35
COMP_G = (4589 / 1024, -16577 / 1024, 25614 / 1024, -12860 / 1024)


class SMCfg:
    """approx.py:38-72 defaults."""

    def __init__(self, base_range=8.0, extension_base=2.0, extension_steps=5, precise=True,
                 exp_range=8, inv_range=100.0, inv_iters=16):
        self.base_range, self.extension_base = base_range, extension_base
        self.extension_steps, self.precise = extension_steps, precise
        self.exp_range, self.inv_range, self.inv_iters = exp_range, inv_range, inv_iters

    @property
    def max_range(self):
        return int(math.ceil(self.base_range * self.extension_base ** self.extension_steps / 2))

    @property
    def dep_delta(self):
        return 4.0 / (27.0 * self.base_range ** 2)


def _is(x):
    return isinstance(x, Grid)


def _add(x, y):
    return x.add(y) if _is(x) else (y.add(x) if _is(y) else x + y)


def _sub(x, y):
    return x.sub(y) if _is(x) else (y.rsub(x) if _is(y) else x - y)


def _mul(x, y):
    return x.mul(y) if _is(x) else (y.mul(x) if _is(y) else x * y)


def _scale(x, t):
    return x.scale(t) if _is(x) else x * t


class _Layout:
    """approx.py:118-189 — layout facts for one softmax input."""

    def __init__(self, M, classes=None, period=None):
        self.enc = _is(M)
        if self.enc:
            if M.tiling != "horizontal" or M.grid[1] != 1:
                raise ShapeMismatch("softmax layout")
            self.classes = M.shape[1] if classes is None else classes
            self.period = M.period if period is None else period
            self.ctx, self.mat = M.ctx, M
        else:
            arr = np.asarray(M, dtype=np.float64)
            self.classes = arr.shape[1] if classes is None else classes
            self.period = npow2(self.classes) if period is None else period
            self.ctx = None
            pad = np.zeros((arr.shape[0], self.period))
            pad[:, :self.classes] = arr[:, :self.classes]
            self.mat = pad

    def pat(self, f):
        if self.enc:
            cols = f(np.arange(self.ctx.grid_cols))
            return pattern(self.ctx, np.broadcast_to(cols, (self.ctx.grid_rows, self.ctx.grid_cols)),
                           self.mat.grid)
        return f(np.arange(self.period))[None, :]

    def keep(self):
        c = self.classes
        return self.pat(lambda j: np.where(j < c, 1.0, 0.0))

    def pad_half(self):
        c, cp = self.classes, self.period
        return self.pat(lambda j: np.where((j % cp) >= c, 0.5, 0.0))

    def first_col(self):
        return self.pat(lambda j: np.where(j == 0, 1.0, 0.0))

    def bcast0(self, x):
        if self.enc:
            return x.each(lambda b: ladder(self.ctx, b, -1, lg(self.ctx.grid_cols)))
        return np.repeat(x[:, :1], self.period, axis=1)

    def rowsum(self, x):
        if self.enc:
            return col_sums(x)
        s = x
        for t in range(lg(self.period)):
            s = s + np.roll(s, -(1 << t), axis=1)
        return np.repeat(s[:, :1], self.period, axis=1)

    def retile(self, x):
        if not self.enc:
            return x
        return x.each(lambda b: ladder(self.ctx, b, -self.period, lg(self.ctx.grid_cols // self.period)))


def _odd7(x, a):                                                    # approx.py:195-202
    y = _mul(x, x)
    acc = _add(_scale(y, a[3]), a[2])
    acc = _add(_mul(acc, y), a[1])
    acc = _add(_mul(acc, y), a[0])
    return _mul(acc, x)


def a_comp(x, y):                                                   # approx.py:205-213
    u = _odd7(_odd7(_odd7(_sub(x, y), COMP_G), COMP_G), COMP_F)
    return _scale(_add(u, 1.0), 0.5)


def a_max(M, cfg, classes=None, period=None):                       # approx.py:216-238
    L = _Layout(M, classes, period)
    two_r = 2.0 * cfg.max_range
    work = _scale(L.mat, 1.0 / two_r)
    if L.classes < L.period:
        work = _sub(work, L.pad_half())
    best = work
    for t in range(lg(L.period)):
        rival = best.lrot(1 << t) if _is(best) else np.roll(best, -(1 << t), axis=1)
        w = a_comp(best, rival)
        best = _add(_mul(best, w), _mul(rival, _sub(1.0, w)))
    best = _mul(best, L.first_col())
    best = L.bcast0(best)
    return _scale(best, two_r)


def domain_extend(M, cfg):                                          # approx.py:241-253
    for i in range(cfg.extension_steps - 1, -1, -1):
        d = cfg.dep_delta * float(cfg.extension_base) ** (-2 * i)
        sq = _mul(M, M)
        sc = _scale(M, d)
        M = _sub(M, _mul(sq, sc))
    return M


def dep_comp(M, cfg):                                               # approx.py:256-273
    L2 = float(cfg.extension_base) ** 2
    Ln = L2 ** cfg.extension_steps
    K = L2 * (Ln - 1.0) / (Ln * (L2 - 1.0))
    R = cfg.base_range
    c3 = 1.0 * (4.0 / 27.0) * K / R ** 2
    c5 = 1.0 * (4.0 / 27.0) * K / R ** 4
    sq = _mul(M, M)
    cube = _mul(sq, M)
    fifth = _mul(cube, sq)
    return _add(M, _sub(_scale(cube, c3), _scale(fifth, c5)))


def a_exp(M, cfg):                                                  # approx.py:276-292
    B = cfg.exp_range
    z = _scale(M, 1.0 / B)
    acc = _add(_scale(z, EXP_POLY[12]), EXP_POLY[11])
    for k in range(10, -1, -1):
        acc = _add(_mul(acc, z), EXP_POLY[k])
    for _ in range(lg(B)):
        acc = _mul(acc, acc)
    return acc


def a_inv(M, cfg):                                                  # approx.py:295-309
    y = _scale(M, 1.0 / cfg.inv_range)
    a = _sub(2.0, y)
    b = _sub(1.0, y)
    for _ in range(cfg.inv_iters):
        b = _mul(b, b)
        a = _mul(a, _add(b, 1.0))
    return _scale(a, 1.0 / cfg.inv_range)


def a_softmax(M, cfg=None, classes=None, period=None):              # approx.py:312-344
    cfg = cfg or SMCfg()
    L = _Layout(M, classes, period)
    work = L.mat
    best = a_max(work if L.enc else work[:, :L.classes], cfg, classes=L.classes, period=L.period)
    keep = L.keep()
    norm = _mul(_sub(work, best), keep)
    norm = domain_extend(norm, cfg)
    if cfg.precise:
        norm = dep_comp(norm, cfg)
    expd = _mul(a_exp(norm, cfg), keep)
    total = L.rowsum(expd)
    recip = a_inv(total, cfg)
    out = L.retile(_mul(expd, recip))
    if L.enc:
        return out.meta((M.shape[0], L.classes), "horizontal", L.period)
    return out[:, :L.classes]


def exact_softmax(z):                                               # plainref.py:21-26
    z = np.asarray(z, dtype=np.float64)
    e = np.exp(z - np.max(z, axis=1, keepdims=True))
    return e / np.sum(e, axis=1, keepdims=True)


# ---------------------------------------------------------------------------
# L3: NAG step (training.py) and the float64 twin (plainref.py)
# ---------------------------------------------------------------------------


class State:
    def __init__(self, weights, momentum, lam=1.0):
        self.weights, self.momentum, self.lam, self.t = weights, momentum, lam, 1


def nag_step(st, X, Y, lr, batch_rows, cfg=None, threshold=5, presum=row_presum):
    """training.py:66-100 (trace hook omitted: it is an observer decode)."""
    cfg = cfg or SMCfg()
    logits = diag_abt(X, st.momentum)
    probs = a_softmax(logits, cfg)
    resid = probs.sub(Y)
    grad = diag_atb(resid, X, scale=lr / batch_rows, presum=presum)
    w_next = st.momentum.sub(grad)
    lam_next = (1.0 + math.sqrt(1.0 + 4.0 * st.lam ** 2)) / 2.0
    gamma = (1.0 - st.lam) / lam_next
    v_next = w_next.scale(1.0 - gamma).add(st.weights.scale(gamma))
    if min(w_next.level, v_next.level) < threshold:
        w_next, v_next = w_next.bootstrap(), v_next.bootstrap()
    st.weights, st.momentum, st.lam, st.t = w_next, v_next, lam_next, st.t + 1
    return logits


def init_weights(classes, dim, seed):                               # plainref.py:50-53
    return np.random.default_rng(seed).uniform(-0.01, 0.01, size=(classes, dim))


def one_hot(labels, classes):
    labels = np.asarray(labels, dtype=int)
    out = np.zeros((labels.shape[0], classes))
    out[np.arange(labels.shape[0]), labels] = 1.0
    return out


def plain_step(W, V, lam, xb, yb, lr, softmax_fn):                  # plainref.py:85-96
    probs = softmax_fn(xb @ V.T)
    grad = (probs - yb).T @ xb * (lr / xb.shape[0])
    w_next = V - grad
    lam_next = (1.0 + math.sqrt(1.0 + 4.0 * lam * lam)) / 2.0
    gamma = (1.0 - lam) / lam_next
    return w_next, (1.0 - gamma) * w_next + gamma * W, lam_next
