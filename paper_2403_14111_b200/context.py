"""``CKKSContext``: the reference backend interface over the B200 CUDA library.

Drop-in for ``hefit.emulator.EmulatorContext`` (emulator.py:111-281): same
attributes (``slot_count``, ``grid_rows``, ``grid_cols``, ``max_level``,
``auto_bootstrap``, ``ledger``, ``decode_events``), same methods
(``encrypt``/``pack``/``add``/``sub``/``mult``/``cmult``/``lrot``/``rrot``/
``conj``/``mul_i``/``bootstrap``/``note_decode``/``decodes_by``), same
operand rules (block, Python/numpy scalar, raw slot array) and the same
ledger increments and level rules.  Ciphertext blocks live in HBM as RNS
residues; ``.slots`` is an audited client-side decrypt.

Differences forced by real CKKS: values carry noise
(decode tolerance ``DECODE_TOL``); operands at different levels are
level-adjusted (unledgered, counted in ``ctx.extra['LevelAdjust']``);
``bootstrap`` is a labelled refresh surrogate, not CKKS bootstrapping.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
import threading

import numpy as np

from . import _native as N
from .errors import DepthExhausted, SlotCountMismatch

OP_KINDS = ("Add", "CMult", "Mult", "Rot", "Conj", "Bootstrap")
EXTRA_KINDS = ("LevelAdjust", "KeySwitch")
DEFAULT_OP_WEIGHTS_MS = {"Add": 0.085, "CMult": 0.9, "Mult": 1.6, "Rot": 1.2, "Conj": 1.2,
                         "Bootstrap": 159.0}
PLAINTEXT_LEVEL = math.inf
DECODE_TOL = 1e-3      # CKKS noise after a full DiagABT/DiagATB at Delta = 2^42 is ~2e-4

# name -> (log N, q bits (q0 first), p bits, alpha, log scale, hamming weight)
PARAMS = {
    # BASELINE config 0: N=2^13, 60 + 4x40 | 60, Delta 2^40
    "cfg0": (13, [60] + [40] * 4, [60], 1, 40, 64),
    # BASELINE configs 1-4: N=2^16, 58 + 12x42 | 3x60, dnum 4, Delta 2^42
    "cfg1": (16, [58] + [42] * 12, [60] * 3, 4, 42, 64),
    # cfg1's chain on a tiny ring (test-only, insecure)
    "small12": (9, [58] + [42] * 12, [60] * 3, 4, 42, 64),
    # cfg1's chain at the reference's default run_steps context
    # (EmulatorContext(4096, 64, max_level=12), training.py:361); insecure ring
    "n13l12": (13, [58] + [42] * 12, [60] * 3, 4, 42, 64),
    # bootstrappable chain: q0 60 bits, 12 application levels
    # of 42 bits (scale 2^42), then 58 / 60 / 15 x 55 bits for SlotToCoeff,
    # EvalMod and CoeffToSlot (top scale 2^55); P = 4 x 60 bits
    "boot16": (16, [60] + [42] * 12 + [58, 60] + [55] * 15, [60] * 4, 4, 55, 64),
    # the same chain on a 2^10 ring (test-only, insecure): bootstrapping parity
    "boot10": (10, [60] + [42] * 12 + [58, 60] + [55] * 15, [60] * 4, 4, 55, 64),
    "tiny": (10, [50] + [40] * 3, [50], 1, 40, 32),
    # short chains on the other split-pass rings (test-only): the fused
    # key-switch / rescale pipeline's column-pass geometries for 2^14, 2^15, 2^17
    "n14": (14, [58] + [42] * 5, [60] * 2, 2, 42, 64),
    "n15": (15, [58] + [42] * 4, [60] * 3, 3, 42, 64),
    "n17": (17, [58] + [42] * 3, [60], 1, 42, 64),
}


# parameter sets whose chain carries bootstrapping levels above the
# application's: the EmulatorContext's max_level is this application level
APP_LEVELS = {"boot16": 12, "boot10": 12}
BOOTSTRAP_MODES = ("surrogate", "ckks")


def params_for(slot_count: int, max_level: int) -> str:
    for name, (logn, qb, _pb, _a, _s, _h) in PARAMS.items():
        if (1 << (logn - 1)) == slot_count and len(qb) - 1 == max_level:
            return name
    raise ValueError(f"no CKKS parameter set with {slot_count} slots and max_level {max_level}")


class NativeLedger:
    """OpLedger interface (emulator.py:70-108) over the library's counters."""

    def __init__(self, ctx: "CKKSContext", weights=None):
        self._ctx = ctx
        self.weights = dict(DEFAULT_OP_WEIGHTS_MS)
        if weights:
            self.weights.update(weights)
        self._offset = dict.fromkeys(OP_KINDS, 0)
        self._lock = threading.Lock()

    def _raw(self):
        arr = (C.c_int64 * N.NCOUNTS)()
        N.check(N.lib().hc_ctx_counts(self._ctx._h, arr, 0))
        return list(arr)

    def record(self, kind: str, n: int = 1) -> None:
        with self._lock:
            self._offset[kind] += n

    def counts(self):
        raw = self._raw()
        with self._lock:
            return {k: raw[i] + self._offset[k] for i, k in enumerate(OP_KINDS)}

    def extra(self):
        raw = self._raw()
        return {k: raw[len(OP_KINDS) + i] for i, k in enumerate(EXTRA_KINDS)}

    snapshot = counts

    def delta(self, before):
        now = self.counts()
        return {k: now[k] - before.get(k, 0) for k in OP_KINDS}

    @property
    def estimated_ms(self) -> float:
        c = self.counts()
        return float(sum(c[k] * self.weights.get(k, 0.0) for k in OP_KINDS))

    def estimate_ms(self, counts) -> float:
        return float(sum(counts.get(k, 0) * self.weights.get(k, 0.0) for k in OP_KINDS))

    def reset(self) -> None:
        N.check(N.lib().hc_ctx_counts(self._ctx._h, None, 1))
        with self._lock:
            self._offset = dict.fromkeys(OP_KINDS, 0)


class PlainBlock:
    """Plaintext block (encrypted=False, level inf): host slots, never ledgered."""

    __slots__ = ("slots", "level", "encrypted", "_key")

    def __init__(self, slots):
        a = np.ascontiguousarray(np.asarray(slots, dtype=np.complex128))
        a.setflags(write=False)
        self.slots, self.level, self.encrypted, self._key = a, PLAINTEXT_LEVEL, False, None

    def __len__(self):
        return int(self.slots.shape[0])

    @property
    def key(self) -> bytes:
        if self._key is None:
            self._key = hashlib.blake2b(self.slots.tobytes(), digest_size=16).hexdigest().encode()
        return self._key


class Ciphertext:
    """A ciphertext block: device residues [2][level+1][N] behind a C handle."""

    __slots__ = ("ctx", "_h", "level", "encrypted", "__weakref__")

    def __init__(self, ctx: "CKKSContext", handle):
        self.ctx = ctx
        self._h = handle
        self.level = int(N.lib().hc_ct_level(handle))
        self.encrypted = True

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                N.lib().hc_ct_free(h)
            except Exception:
                pass
            self._h = None

    def __len__(self):
        return self.ctx.slot_count

    @property
    def slots(self) -> np.ndarray:
        """Client-side decrypt + decode (the audited path behind decode())."""
        return self.ctx.decrypt(self)

    def residues(self) -> np.ndarray:
        out = np.zeros((2, self.level + 1, self.ctx.N), np.uint64)
        N.check(N.lib().hc_ct_download(self._h, out.ctypes.data_as(N.U64P)))
        return out


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(N.DP)


class CKKSContext:
    """EmulatorContext duck type over RNS-CKKS on a B200."""

    def __init__(self, params: str | int = "cfg1", grid_rows: int | None = None, *, max_level=None,
                 auto_bootstrap: bool = False, seed: int = 2024, sigma: float = 3.2, device: int = 0,
                 op_weights=None, hoist: bool = True, bootstrap: str = "surrogate"):
        if isinstance(params, (int, np.integer)):
            params = params_for(int(params), 12 if max_level is None else max_level)
        logn, qb, pb, alpha, logs, hw = PARAMS[params]
        self.params = params
        self.logN, self.N = logn, 1 << logn
        self.slot_count = self.N // 2
        if grid_rows is None:
            grid_rows = 1 << ((logn - 1) // 2)
        if grid_rows < 1 or grid_rows & (grid_rows - 1) or grid_rows > self.slot_count:
            raise SlotCountMismatch(f"grid_rows must be a power of two <= slot_count, got {grid_rows}")
        self.grid_rows = grid_rows
        self.grid_cols = self.slot_count // grid_rows
        self.max_level = APP_LEVELS.get(params, len(qb) - 1)
        self.chain_top = len(qb) - 1
        if max_level is not None and max_level != self.max_level:
            raise ValueError(f"parameter set {params} has max_level {self.max_level}")
        self.K, self.alpha = len(pb), alpha
        self.dnum = -(-len(qb) // alpha)
        self.seed = seed
        h = C.c_void_p()
        qa = (C.c_int * len(qb))(*qb)
        pa = (C.c_int * len(pb))(*pb)
        N.check(N.lib().hc_ctx_create(logn, len(qb), qa, len(pb), pa, alpha, logs, hw, sigma, seed, device,
                                      C.byref(h)))
        self._h = h
        N.check(N.lib().hc_set_grid_rows(self._h, grid_rows))
        if self.max_level != self.chain_top:
            N.check(N.lib().hc_set_app_level(self._h, self.max_level))
        if bootstrap not in BOOTSTRAP_MODES:
            raise ValueError(f"bootstrap must be one of {BOOTSTRAP_MODES}")
        self.bootstrap_mode = bootstrap
        N.check(N.lib().hc_set_bootstrap(self._h, int(bootstrap == "ckks")))
        self._auto = False
        self.auto_bootstrap = auto_bootstrap
        self._hoist = True
        self.hoist = hoist
        self.ledger = NativeLedger(self, op_weights)
        self.decode_events: list = []
        n = len(qb) + len(pb)
        self.moduli = np.zeros(n, np.uint64)
        self.scales = np.zeros(len(qb))
        N.check(N.lib().hc_ctx_info(self._h, self.moduli.ctypes.data_as(N.U64P), _dptr(self.scales)))

    def __del__(self):
        # ciphertexts hold a strong reference to their context, so none is alive here
        self.close()

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            try:
                N.lib().hc_ctx_destroy(h)
            except Exception:
                pass

    # -- settings ----------------------------------------------------------
    @property
    def auto_bootstrap(self) -> bool:
        return self._auto

    @auto_bootstrap.setter
    def auto_bootstrap(self, on: bool) -> None:
        self._auto = bool(on)
        N.check(N.lib().hc_set_auto_bootstrap(self._h, int(self._auto)))

    @property
    def hoist(self) -> bool:
        """Fused schedule forms: hoisted rotations and one
        relinearisation per product sum, in the native schedules and through
        ``lrot_hoisted`` / ``mult_sum``.  The oracle context's ``hoist`` must
        match for residue parity; the ledger is the reference's either way."""
        return self._hoist

    @hoist.setter
    def hoist(self, on: bool) -> None:
        self._hoist = bool(on)
        N.check(N.lib().hc_set_hoist(self._h, int(self._hoist)))

    @property
    def extra(self):
        return self.ledger.extra()

    def set_streams(self, n: int) -> None:
        """Fan-out of the native schedules' independent diagonal passes (1 = serial)."""
        N.check(N.lib().hc_set_streams(self._h, int(n)))

    @property
    def nonce(self) -> int:
        v = C.c_uint64()
        N.check(N.lib().hc_ctx_nonce(self._h, C.byref(v), None))
        return v.value

    @nonce.setter
    def nonce(self, n: int) -> None:
        v = C.c_uint64(n)
        N.check(N.lib().hc_ctx_nonce(self._h, None, C.byref(v)))

    def _next_nonce(self) -> int:
        n = self.nonce
        self.nonce = n + 1
        return n

    def sync(self):
        N.check(N.lib().hc_sync(self._h))

    def model_bytes(self, reset: bool = False) -> float:
        """SURVEY §8(d) per-op HBM model (bytes) of the ledgered ops so far."""
        v = C.c_double()
        N.check(N.lib().hc_ctx_model_bytes(self._h, C.byref(v), int(reset)))
        return v.value

    def set_shard(self, total_blocks: int, first_block: int) -> None:
        """Block-row sharding: this context holds block rows
        ``first_block ..`` of a batch of ``total_blocks``; the softmax's refresh
        nonces then follow the whole batch's sequential order (``hc_set_shard``)."""
        N.check(N.lib().hc_set_shard(self._h, int(total_blocks), int(first_block)))

    def set_pass_shard(self, world: int, rank: int, reducer=None) -> None:
        """Diagonal-pass sharding of diag_abt / diag_atb (``hc_set_pass_shard``):
        this context runs passes k = rank (mod world); ``reducer(ctx, handles)``
        replaces the partial accumulators by their modular sum over ranks."""
        if world > 1 and reducer is None:
            raise ValueError("pass sharding needs a reducer")
        if world > 1:
            from .matmul import _reduce_callback
            self._pass_cb = _reduce_callback(self, reducer)
        else:
            self._pass_cb = N.REDUCE_FN(0)
        N.check(N.lib().hc_set_pass_shard(self._h, int(world), int(rank), self._pass_cb, None))

    def stream(self) -> int:
        """The cudaStream_t the library issues on right now (for stream handoff)."""
        s = C.c_void_p()
        N.check(N.lib().hc_ctx_stream(self._h, C.byref(s)))
        return int(s.value or 0)

    def mod_reduce(self, ct) -> None:
        """Finish a cross-rank uint64 sum held in ``ct``'s residues, in place (K8)."""
        N.check(N.lib().hc_mod_reduce(self._h, ct._h if isinstance(ct, Ciphertext) else ct))

    def keygen(self, galois: int):
        N.check(N.lib().hc_keygen(self._h, int(galois)))

    def galois_rot(self, r: int) -> int:
        return int(N.lib().hc_galois_rot(self._h, int(r)))

    def rotation_keys(self, steps):
        for r in steps:
            if int(r) % self.slot_count:
                self.keygen(self.galois_rot(r))

    # -- construction ------------------------------------------------------
    def _vec(self, values) -> np.ndarray:
        a = np.asarray(values, dtype=np.complex128).ravel()
        if a.shape[0] != self.slot_count:
            raise SlotCountMismatch(f"expected {self.slot_count} slots, got {a.shape[0]}")
        return a

    def encrypt(self, values, level: int | None = None) -> Ciphertext:
        lv = self.max_level if level is None else level
        if not 0 <= lv <= self.max_level:
            raise ValueError(f"level must be in [0, {self.max_level}], got {lv}")
        v = self._vec(values)
        re, im = np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag)
        h = C.c_void_p()
        N.check(N.lib().hc_encrypt(self._h, _dptr(re), _dptr(im), lv, self._next_nonce(), C.byref(h)))
        return Ciphertext(self, h)

    def pack(self, values) -> PlainBlock:
        return PlainBlock(self._vec(values))

    def decrypt(self, ct: Ciphertext) -> np.ndarray:
        re = np.zeros(self.slot_count)
        im = np.zeros(self.slot_count)
        N.check(N.lib().hc_decrypt(self._h, ct._h, _dptr(re), _dptr(im)))
        return re + 1j * im

    def from_residues(self, residues: np.ndarray, level: int) -> Ciphertext:
        a = np.ascontiguousarray(residues, dtype=np.uint64)
        if a.shape != (2, level + 1, self.N):
            raise ValueError(f"residues must be (2, {level + 1}, {self.N})")
        h = C.c_void_p()
        N.check(N.lib().hc_ct_upload(self._h, a.ctypes.data_as(N.U64P), level, C.byref(h)))
        return Ciphertext(self, h)

    def encode_pt(self, values, level: int) -> np.ndarray:
        """Residues of a plaintext encoded at scales[level] (parity helper)."""
        v = self._vec(values)
        re, im = np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag)
        h = C.c_void_p()
        N.check(N.lib().hc_encode_pt(self._h, _dptr(re), _dptr(im), level, C.byref(h)))
        out = np.zeros((level + 1, self.N), np.uint64)
        try:
            N.check(N.lib().hc_pt_download(h, out.ctypes.data_as(N.U64P)))
        finally:
            N.lib().hc_pt_free(h)
        return out

    def encode_coef(self, values, scale: float) -> np.ndarray:
        v = self._vec(values)
        re, im = np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag)
        out = np.zeros(self.N, np.int64)
        N.check(N.lib().hc_encode_coef(self._h, _dptr(re), _dptr(im), float(scale), out.ctypes.data_as(N.I64P)))
        return out

    def key(self, galois: int) -> np.ndarray:
        out = np.zeros((self.dnum, 2, len(self.moduli), self.N), np.uint64)
        N.check(N.lib().hc_key_download(self._h, int(galois), out.ctypes.data_as(N.U64P)))
        return out

    # -- operand plumbing (emulator.py:172-182) -----------------------------
    def _kind(self, v):
        if isinstance(v, Ciphertext):
            if v.ctx is not self:
                raise SlotCountMismatch("ciphertext from another context")
            return "ct", v
        if isinstance(v, PlainBlock):
            if len(v) != self.slot_count:
                raise SlotCountMismatch(f"block has {len(v)} slots, context expects {self.slot_count}")
            return "vec", v
        if hasattr(v, "slots") and hasattr(v, "encrypted") and not v.encrypted:
            return "vec", PlainBlock(self._vec(v.slots))
        if isinstance(v, (int, float, complex, np.integer, np.floating, np.complexfloating)):
            return "scalar", complex(v)
        return "vec", PlainBlock(self._vec(v))

    def _new(self, fn, *args) -> Ciphertext:
        h = C.c_void_p()
        N.check(fn(self._h, *args, C.byref(h)))
        return Ciphertext(self, h)

    def _plain_args(self, pb: PlainBlock):
        re = np.ascontiguousarray(pb.slots.real)
        im = np.ascontiguousarray(pb.slots.imag)
        return re, im, pb.key

    # -- arithmetic (emulator.py:195-273) ----------------------------------
    def _addsub(self, x, y, sub: bool):
        kx, vx = self._kind(x)
        ky, vy = self._kind(y)
        L = N.lib()
        if kx != "ct" and ky != "ct":
            ax = vx if kx == "scalar" else vx.slots
            ay = vy if ky == "scalar" else vy.slots
            return PlainBlock(np.broadcast_to(ax - ay if sub else ax + ay, (self.slot_count,)))
        if kx == "ct" and ky == "ct":
            return self._new(L.hc_op_add, vx._h, vy._h, int(sub))
        if kx == "ct":
            ct, other, kother, mode = vx, vy, ky, (1 if sub else 0)
        else:
            ct, other, kother, mode = vy, vx, kx, (2 if sub else 0)
        if kother == "scalar":
            return self._new(L.hc_op_add_scalar, ct._h, other.real, other.imag, mode)
        re, im, key = self._plain_args(other)
        return self._new(L.hc_op_add_plain, ct._h, _dptr(re), _dptr(im), key, mode)

    def add(self, x, y):
        return self._addsub(x, y, False)

    def sub(self, x, y):
        return self._addsub(x, y, True)

    def mult(self, x, y):
        kx, vx = self._kind(x)
        ky, vy = self._kind(y)
        L = N.lib()
        if kx == "ct" and ky == "ct":
            return self._new(L.hc_op_mult, vx._h, vy._h)
        if kx != "ct" and ky != "ct":
            ax = vx if kx == "scalar" else vx.slots
            ay = vy if ky == "scalar" else vy.slots
            return PlainBlock(np.broadcast_to(ax * ay, (self.slot_count,)))
        ct, other, kother = (vx, vy, ky) if kx == "ct" else (vy, vx, kx)
        if kother == "scalar":
            return self._new(L.hc_op_mult_scalar, ct._h, other.real, other.imag)
        re, im, key = self._plain_args(other)
        return self._new(L.hc_op_mult_plain, ct._h, _dptr(re), _dptr(im), key)

    def cmult(self, x, y):
        if isinstance(y, Ciphertext):
            raise TypeError("cmult expects a plaintext second operand")
        return self.mult(x, y)

    def lrot(self, x, r: int):
        kx, vx = self._kind(x)
        r = int(r) % self.slot_count
        if r == 0:
            return x if isinstance(x, (Ciphertext, PlainBlock)) else vx
        if kx != "ct":
            return PlainBlock(np.roll(vx.slots if kx == "vec" else np.full(self.slot_count, vx), -r))
        return self._new(N.lib().hc_op_lrot, vx._h, r)

    def rrot(self, x, r: int):
        return self.lrot(x, -int(r))

    def lrot_hoisted(self, x, rs):
        """[lrot(x, r) for r in rs] with one shared ModUp (hoisted rotations):
        one Rot per non-zero r, r = 0 returns x itself."""
        kx, vx = self._kind(x)
        rr = [int(r) % self.slot_count for r in rs]
        if kx != "ct" or not self._hoist:
            return [self.lrot(x, r) for r in rr]
        arr = (C.c_int64 * len(rr))(*rr)
        outs = (C.c_void_p * len(rr))()
        N.check(N.lib().hc_op_lrot_hoisted(self._h, vx._h, arr, len(rr), outs))
        res = []
        for r, h in zip(rr, outs):
            if r == 0:
                N.lib().hc_ct_free(h)
                res.append(x)
            else:
                res.append(Ciphertext(self, C.c_void_p(h)))
        return res

    def ladder(self, x, stride: int, steps: int):
        """The reference's doubling ladder ``for t < steps: x = add(x, lrot(x,
        stride * 2^t))`` (encoding.py:354-359, 378-379; stride < 0: rrot):
        steps Rot + steps Add on the ledger.  With ``hoist`` on, two steps run
        as one radix-4 rotate-and-sum stage (one ModUp, one ModDown)."""
        kx, vx = self._kind(x)
        if kx != "ct":
            for t in range(int(steps)):
                x = self.add(x, self.lrot(x, int(stride) * (1 << t)))
            return x
        return self._new(N.lib().hc_op_ladder, vx._h, int(stride), int(steps))

    def mult_sum(self, xs, ys):
        """add(...add(mult(x0, y0), mult(x1, y1))...) with one relinearisation
        and rescale (n Mult + n - 1 Add on the ledger) when every operand is a
        ciphertext at one level >= 1 and n >= 2; the separate ops otherwise."""
        xs, ys = list(xs), list(ys)
        blocks = xs + ys
        if (not self._hoist or len(xs) < 2 or not all(isinstance(b, Ciphertext) for b in blocks)
                or len({b.level for b in blocks}) != 1 or blocks[0].level < 1):
            acc = self.mult(xs[0], ys[0])
            for x, y in zip(xs[1:], ys[1:]):
                acc = self.add(acc, self.mult(x, y))
            return acc
        A = (C.c_void_p * len(xs))(*[x._h for x in xs])
        B = (C.c_void_p * len(ys))(*[y._h for y in ys])
        return self._new(N.lib().hc_op_mult_sum, A, B, len(xs))

    def conj(self, x):
        kx, vx = self._kind(x)
        if kx != "ct":
            return PlainBlock(np.conj(vx.slots if kx == "vec" else np.full(self.slot_count, vx)))
        return self._new(N.lib().hc_op_conj, vx._h)

    def mul_i(self, x):
        kx, vx = self._kind(x)
        if kx != "ct":
            return PlainBlock((vx.slots if kx == "vec" else np.full(self.slot_count, vx)) * 1j)
        return self._new(N.lib().hc_op_mul_i, vx._h)

    def bootstrap(self, x):
        if not isinstance(x, Ciphertext):
            return x
        return self._new(N.lib().hc_op_bootstrap, x._h)

    # exact primitives (no ledger)
    def ckks_bootstrap(self, x: Ciphertext) -> Ciphertext:
        """One CKKS bootstrapping, whatever ``bootstrap_mode`` is."""
        return self._new(N.lib().hc_bootstrap_ct, x._h)

    def rescale(self, x: Ciphertext) -> Ciphertext:
        return self._new(N.lib().hc_rescale, x._h)

    def level_adjust(self, x: Ciphertext, level: int) -> Ciphertext:
        return self._new(N.lib().hc_level_adjust, x._h, int(level))

    # -- audit (emulator.py:277-281) ------------------------------------------
    def note_decode(self, role: str, tag=None) -> None:
        self.decode_events.append((role, tag))

    def decodes_by(self, role: str):
        return [ev for ev in self.decode_events if ev[0] == role]
