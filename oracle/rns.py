"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over the C RNS-CKKS oracle and an
``EmulatorContext``-duck-typed context on top of it.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this.  ``OracleCKKSContext`` restates, over real RNS-CKKS residues,
the op semantics of the reference backend (``emulator.py:111-281``): level
rules, auto-bootstrap per operand (``emulator.py:184-191``), the ledger
(``emulator.py:70-108``), ``lrot`` by 0 returning the same object
(``emulator.py:244-245``).  The CKKS-specific policy — per-level canonical
scales, level adjustment when operand levels differ, refresh surrogate — is
the one DESIGN.md §3 pins and the CUDA product implements.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess

import numpy as np

from . import slots as S

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "libckks_oracle.so")

# parameter sets with bootstrapping levels above the application's top level
APP_LEVELS = {"boot16": 12, "boot10": 12}

# name -> (logN, q bits, p bits, alpha, log scale, hamming weight)
PARAMS = {
    "cfg0": (13, [60] + [40] * 4, [60], 1, 40, 64),
    "cfg1": (16, [58] + [42] * 12, [60] * 3, 4, 42, 64),
    # cfg1's modulus chain on a tiny ring: deep schedules (softmax, NAG step)
    # in milliseconds; not secure, test-only
    "small12": (9, [58] + [42] * 12, [60] * 3, 4, 42, 64),
    # the same chain at the reference's default training ring (2^13 slots x 2)
    "n13l12": (13, [58] + [42] * 12, [60] * 3, 4, 42, 64),
    # bootstrappable chain: q0 60 bits, 12 application levels
    # of 42 bits, then 58 / 60 / 15 x 55 bits for SlotToCoeff, EvalMod and
    # CoeffToSlot; P = 4 x 60 bits; top scale 2^55 (scale 2^42 from level 12 down)
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


def build():
    subprocess.check_call(["make", "-s", "-C", HERE], stdout=subprocess.DEVNULL)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        P, U, I, D = C.c_void_p, C.c_uint64, C.c_int, C.c_double
        ptr = np.ctypeslib.ndpointer
        u64p = ptr(np.uint64, flags="C_CONTIGUOUS")
        i64p = ptr(np.int64, flags="C_CONTIGUOUS")
        f64p = ptr(np.float64, flags="C_CONTIGUOUS")
        L.orc_create.restype = P
        L.orc_create.argtypes = [I, I, C.POINTER(I), I, C.POINTER(I), I, I, I, D, U]
        L.orc_destroy.argtypes = [P]
        L.orc_info.argtypes = [P, u64p, f64p, u64p]
        L.orc_secret.argtypes = [P, i64p]
        L.orc_cdt.argtypes = [P, u64p]
        L.orc_encode.argtypes = [P, f64p, f64p, D, i64p]
        L.orc_decode_real.argtypes = [P, f64p, f64p, f64p]
        L.orc_encrypt.argtypes = [P, f64p, f64p, I, U, u64p]
        L.orc_encrypt_coef.argtypes = [P, i64p, I, U, u64p]
        L.orc_encode_ntt.argtypes = [P, f64p, f64p, I, D, u64p]
        L.orc_decrypt.argtypes = [P, u64p, I, f64p, f64p]
        L.orc_refresh.argtypes = [P, u64p, I, U, u64p]
        L.orc_add.argtypes = [P, u64p, u64p, I, I, I, u64p]
        L.orc_neg.argtypes = [P, u64p, I, u64p]
        L.orc_add_const.argtypes = [P, u64p, I, D, D, u64p]
        L.orc_mul_const.argtypes = [P, u64p, I, D, D, u64p]
        L.orc_mul_i.argtypes = [P, u64p, I, u64p]
        L.orc_mul_pt.argtypes = [P, u64p, u64p, I, u64p]
        L.orc_mul_pt_raw.argtypes = [P, u64p, u64p, I, u64p]
        L.orc_mul_int.argtypes = [P, u64p, I, U, u64p]
        L.orc_mod_raise.argtypes = [P, u64p, I, u64p]
        L.orc_set_app_level.argtypes = [P, I]
        L.orc_add_pt.argtypes = [P, u64p, u64p, I, I, u64p]
        L.orc_rescale.argtypes = [P, u64p, I, I, u64p]
        L.orc_drop.argtypes = [P, u64p, I, I, u64p]
        L.orc_level_adjust.argtypes = [P, u64p, I, I, u64p]
        L.orc_automorph.argtypes = [P, u64p, I, U, u64p]
        L.orc_galois_rot.restype = U
        L.orc_galois_rot.argtypes = [P, C.c_int64]
        L.orc_mult.argtypes = [P, u64p, u64p, I, u64p]
        L.orc_rotate_hoisted.argtypes = [P, u64p, I, u64p, I, u64p]
        L.orc_mult_sum.argtypes = [P, u64p, u64p, I, I, u64p]
        L.orc_rotsum.argtypes = [P, u64p, I, u64p, I, u64p]
        L.orc_key.argtypes = [P, I, u64p]
        L.orc_ntt_limb.argtypes = [P, I, u64p, I]
        L.orc_mulmod.restype = U
        L.orc_mulmod.argtypes = [P, I, U, U]
        L.orc_rng.restype = U
        L.orc_rng.argtypes = [U, U, U]
        _lib = L
    return _lib


class RnsParams:
    """Raw oracle handle: moduli, scales, encode/decode and per-op residue calls."""

    def __init__(self, name="cfg0", seed=2024, sigma=3.2):
        logN, qb, pb, alpha, logs, hw = PARAMS[name]
        self.name, self.logN, self.N = name, logN, 1 << logN
        self.L, self.K, self.alpha = len(qb) - 1, len(pb), alpha
        self.dnum = -(-len(qb) // alpha)
        self.slots = self.N // 2
        self.app_L = self.L
        qa = (C.c_int * len(qb))(*qb)
        pa = (C.c_int * len(pb))(*pb)
        self.h = lib().orc_create(logN, len(qb), qa, len(pb), pa, alpha, logs, hw, sigma, seed)
        n = len(qb) + len(pb)
        self.moduli = np.zeros(n, np.uint64)
        self.scales = np.zeros(self.L + 1)
        self.psis = np.zeros(n, np.uint64)
        lib().orc_info(self.h, self.moduli, self.scales, self.psis)

    def __del__(self):
        try:
            lib().orc_destroy(self.h)
        except Exception:
            pass

    def ct_shape(self, level):
        return (2, level + 1, self.N)

    def z(self, values):
        v = np.asarray(values, dtype=np.complex128).ravel()
        return np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag)

    def encode(self, values, scale):
        zr, zi = self.z(values)
        out = np.zeros(self.N, np.int64)
        if lib().orc_encode(self.h, zr, zi, float(scale), out) != 0:
            raise OverflowError("encode overflow")
        return out

    def encode_ntt(self, values, level, scale=None):
        zr, zi = self.z(values)
        out = np.zeros((level + 1, self.N), np.uint64)
        if lib().orc_encode_ntt(self.h, zr, zi, level, float(self.scales[level] if scale is None else scale), out):
            raise OverflowError("encode overflow")
        return out

    def encrypt(self, values, level, nonce):
        zr, zi = self.z(values)
        out = np.zeros(self.ct_shape(level), np.uint64)
        if lib().orc_encrypt(self.h, zr, zi, level, nonce, out):
            raise OverflowError("encode overflow")
        return out

    def decrypt(self, ct, level):
        zr = np.zeros(self.slots)
        zi = np.zeros(self.slots)
        lib().orc_decrypt(self.h, np.ascontiguousarray(ct), level, zr, zi)
        return zr + 1j * zi

    def _out(self, level):
        return np.zeros(self.ct_shape(level), np.uint64)

    def add(self, a, b, level, negate=False):
        o = self._out(level)
        lib().orc_add(self.h, a, b, level, 2, int(negate), o)
        return o

    def add_pt(self, a, pt, level, negate=False):
        o = self._out(level)
        lib().orc_add_pt(self.h, a, np.ascontiguousarray(pt), level, int(negate), o)
        return o

    def neg(self, a, level):
        o = self._out(level)
        lib().orc_neg(self.h, a, level, o)
        return o

    def add_const(self, a, level, c):
        o = self._out(level)
        c = complex(c)
        lib().orc_add_const(self.h, a, level, c.real, c.imag, o)
        return o

    def mul_const(self, a, level, c):
        o = self._out(level - 1)
        c = complex(c)
        lib().orc_mul_const(self.h, a, level, c.real, c.imag, o)
        return o

    def mul_pt(self, a, pt, level):
        o = self._out(level - 1)
        lib().orc_mul_pt(self.h, a, np.ascontiguousarray(pt), level, o)
        return o

    def mul_pt_raw(self, a, pt, level):
        o = self._out(level)
        lib().orc_mul_pt_raw(self.h, np.ascontiguousarray(a), np.ascontiguousarray(pt), level, o)
        return o

    def mul_int(self, a, level, k):
        o = self._out(level)
        lib().orc_mul_int(self.h, np.ascontiguousarray(a), level, int(k), o)
        return o

    def mod_raise(self, a, to):
        o = self._out(to)
        lib().orc_mod_raise(self.h, np.ascontiguousarray(a), to, o)
        return o

    def mul_i(self, a, level):
        o = self._out(level)
        lib().orc_mul_i(self.h, a, level, o)
        return o

    def mult(self, a, b, level):
        o = self._out(level - 1)
        lib().orc_mult(self.h, a, b, level, o)
        return o

    def rotate_hoisted(self, a, level, gs):
        o = np.zeros((len(gs),) + self.ct_shape(level), np.uint64)
        lib().orc_rotate_hoisted(self.h, a, level, np.asarray(gs, np.uint64), len(gs), o)
        return list(o)

    def rotsum(self, a, level, gs):
        o = self._out(level)
        lib().orc_rotsum(self.h, a, level, np.asarray(gs, np.uint64), len(gs), o)
        return o

    def mult_sum(self, As, Bs, level):
        o = self._out(level - 1)
        lib().orc_mult_sum(self.h, np.ascontiguousarray(np.stack(As)), np.ascontiguousarray(np.stack(Bs)),
                           len(As), level, o)
        return o

    def rescale(self, a, level):
        o = self._out(level - 1)
        lib().orc_rescale(self.h, np.ascontiguousarray(a), level, a.shape[0], o)
        return o

    def level_adjust(self, a, frm, to):
        o = self._out(to)
        lib().orc_level_adjust(self.h, a, frm, to, o)
        return o

    def galois(self, r):
        return int(lib().orc_galois_rot(self.h, int(r)))

    def automorph(self, a, level, g):
        o = self._out(level)
        lib().orc_automorph(self.h, a, level, g, o)
        return o

    def set_app_level(self, level):
        self.app_L = level
        lib().orc_set_app_level(self.h, level)

    def refresh(self, a, level, nonce):
        o = self._out(self.app_L)
        lib().orc_refresh(self.h, a, level, nonce, o)
        return o

    def secret(self):
        s = np.zeros(self.N, np.int64)
        lib().orc_secret(self.h, s)
        return s

    def key(self, gid):
        out = np.zeros((self.dnum, 2, self.L + 1 + self.K, self.N), np.uint64)
        lib().orc_key(self.h, gid, out)
        return out

    def ntt(self, limb, a, inverse=False):
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().orc_ntt_limb(self.h, limb, a, int(inverse))
        return a


# ---------------------------------------------------------------------------
# EmulatorContext duck type over the oracle
# ---------------------------------------------------------------------------


class RnsBlock:
    """A ciphertext block: residues [2][level+1][N] plus its level."""

    __slots__ = ("ctx", "data", "level", "encrypted")

    def __init__(self, ctx, data, level):
        self.ctx, self.data, self.level, self.encrypted = ctx, data, level, True

    def __len__(self):
        return self.ctx.slot_count

    @property
    def slots(self):
        return self.ctx.p.decrypt(self.data, self.level)


class OracleCKKSContext:
    """EmulatorContext duck type (emulator.py:111-281) over RNS-CKKS residues."""

    def __init__(self, params="cfg0", grid_rows=None, *, auto_bootstrap=False, seed=2024, hoist=True,
                 bootstrap="surrogate"):
        self.p = params if isinstance(params, RnsParams) else RnsParams(params, seed=seed)
        if self.p.name in APP_LEVELS:
            self.p.set_app_level(APP_LEVELS[self.p.name])
        # the reference's bootstrap: the refresh surrogate, or CKKS
        # bootstrapping restated in oracle/boot.py (a nonce is drawn either way)
        self.bootstrap_mode = bootstrap
        self._boot = None
        # fused schedule forms (hoisted rotations, one relinearisation per
        # product sum) where the restated DiagABT / DiagATB use them; the
        # CUDA product's `hoist` flag must match for residue parity
        self.hoist = hoist
        self.slot_count = self.p.slots
        self.grid_rows = grid_rows or (1 << (int(np.log2(self.slot_count)) // 2))
        self.grid_cols = self.slot_count // self.grid_rows
        self.max_level = self.p.app_L
        self.auto_bootstrap = auto_bootstrap
        self.ledger = S.Ledger()
        self.extra = {"LevelAdjust": 0, "KeySwitch": 0}
        self.decode_events = []
        self.nonce = 0
        self._pt = {}

    # -- construction -----------------------------------------------------
    def _vec(self, v):
        a = np.asarray(v, dtype=np.complex128).ravel()
        if a.shape[0] != self.slot_count:
            raise S.SlotCountMismatch(f"expected {self.slot_count} slots, got {a.shape[0]}")
        return a

    def _next_nonce(self):
        n = self.nonce
        self.nonce += 1
        return n

    def encrypt(self, values, level=None):
        lv = self.max_level if level is None else level
        if not 0 <= lv <= self.max_level:
            raise ValueError(f"level must be in [0, {self.max_level}], got {lv}")
        return RnsBlock(self, self.p.encrypt(self._vec(values), lv, self._next_nonce()), lv)

    def pack(self, values):
        return S.Slots(self._vec(values), S.PLAIN_LEVEL, False)

    # -- plumbing ---------------------------------------------------------
    def _kind(self, v):
        if isinstance(v, RnsBlock):
            return "ct", v
        if isinstance(v, S.Slots):
            if len(v) != self.slot_count:
                raise S.SlotCountMismatch("width")
            return "vec", v.slots
        if isinstance(v, (int, float, complex, np.integer, np.floating, np.complexfloating)):
            return "scalar", complex(v)
        return "vec", self._vec(v)

    def _pt_ntt(self, vec, level):
        key = (hashlib.blake2b(np.ascontiguousarray(vec).tobytes(), digest_size=16).digest(), level)
        pt = self._pt.get(key)
        if pt is None:
            pt = self.p.encode_ntt(vec, level)
            self._pt[key] = pt
        return pt

    def _at(self, b, level):
        if b.level == level:
            return b.data
        self.extra["LevelAdjust"] += 1
        return self.p.level_adjust(b.data, b.level, level)

    def _ready(self, b):
        if b.level >= 1:
            return b
        if self.auto_bootstrap:
            self.ledger.record("Bootstrap")
            return self._refresh(b)
        raise S.DepthExhausted(f"mult: operand at level {b.level}")

    def _refresh(self, b):
        nonce = self._next_nonce()
        if self.bootstrap_mode == "ckks":
            if self._boot is None:
                from . import boot
                self._boot = boot.Bootstrapper(self.p, self.max_level)
            return RnsBlock(self, self._boot.bootstrap(b.data, b.level), self.max_level)
        return RnsBlock(self, self.p.refresh(b.data, b.level, nonce), self.max_level)

    # -- arithmetic -------------------------------------------------------
    def _addsub(self, x, y, neg):
        kx, vx = self._kind(x)
        ky, vy = self._kind(y)
        if kx != "ct" and ky != "ct":
            return S.Slots(vx - vy if neg else vx + vy, S.PLAIN_LEVEL, False)
        self.ledger.record("Add")
        if kx == "ct" and ky == "ct":
            lv = min(vx.level, vy.level)
            return RnsBlock(self, self.p.add(self._at(vx, lv), self._at(vy, lv), lv, neg), lv)
        if kx == "ct":
            ct, other, kother, flip = vx, vy, ky, False
        else:
            ct, other, kother, flip = vy, vx, kx, neg   # plain - ct = -(ct) + plain
        lv = ct.level
        d = self.p.neg(ct.data, lv) if flip else ct.data
        sign = -1.0 if (neg and not flip) else 1.0
        if kother == "scalar":
            return RnsBlock(self, self.p.add_const(d, lv, sign * other), lv)
        pt = self._pt_ntt(other, lv)
        return RnsBlock(self, self.p.add_pt(d, pt, lv, negate=(sign < 0)), lv)

    def add(self, x, y):
        return self._addsub(x, y, False)

    def sub(self, x, y):
        return self._addsub(x, y, True)

    def mult(self, x, y):
        kx, vx = self._kind(x)
        ky, vy = self._kind(y)
        if kx == "ct":
            vx = self._ready(vx)
        if ky == "ct":
            vy = self._ready(vy)
        if kx == "ct" and ky == "ct":
            self.ledger.record("Mult")
            self.extra["KeySwitch"] += 1
            lv = min(vx.level, vy.level)
            return RnsBlock(self, self.p.mult(self._at(vx, lv), self._at(vy, lv), lv), lv - 1)
        if kx != "ct" and ky != "ct":
            return S.Slots(vx * vy, S.PLAIN_LEVEL, False)
        self.ledger.record("CMult")
        ct, other, kother = (vx, vy, ky) if kx == "ct" else (vy, vx, kx)
        lv = ct.level
        if kother == "scalar":
            return RnsBlock(self, self.p.mul_const(ct.data, lv, other), lv - 1)
        return RnsBlock(self, self.p.mul_pt(ct.data, self._pt_ntt(other, lv), lv), lv - 1)

    def cmult(self, x, y):
        if isinstance(y, RnsBlock):
            raise TypeError("cmult expects a plaintext second operand")
        return self.mult(x, y)

    def lrot(self, x, r):
        kx, vx = self._kind(x)
        r = int(r) % self.slot_count
        if r == 0:
            return x if isinstance(x, (RnsBlock, S.Slots)) else S.Slots(vx, S.PLAIN_LEVEL, False)
        if kx != "ct":
            return S.Slots(np.roll(vx, -r), S.PLAIN_LEVEL, False)
        self.ledger.record("Rot")
        self.extra["KeySwitch"] += 1
        return RnsBlock(self, self.p.automorph(vx.data, vx.level, self.p.galois(r)), vx.level)

    def rrot(self, x, r):
        return self.lrot(x, -int(r))

    def lrot_hoisted(self, x, rs):
        """lrot(x, r) for every r in rs with one shared ModUp (DESIGN.md §3,
        hoisted rotations): same ledger as the separate calls, r = 0 returns x."""
        kx, vx = self._kind(x)
        rr = [int(r) % self.slot_count for r in rs]
        if kx != "ct":
            return [self.lrot(x, r) for r in rr]
        moving = [r for r in rr if r]
        outs = {}
        if moving:
            self.ledger.record("Rot", len(moving))
            self.extra["KeySwitch"] += len(moving)
            data = self.p.rotate_hoisted(vx.data, vx.level, [self.p.galois(r) for r in moving])
            outs = {r: RnsBlock(self, d, vx.level) for r, d in zip(moving, data)}
        return [outs[r] if r else x for r in rr]

    def rotsum(self, x, rs, steps):
        """x + sum_r lrot(x, r) as one rotate-and-sum stage (DESIGN.md §3,
        radix ladders): one ModUp, the rotations' key products summed in the
        extended basis, one ModDown.  It stands for `steps` doubling steps
        add(x, lrot(x, .)) of the reference's ladder, whose `steps` Rot and
        `steps` Add the ledger records."""
        kx, vx = self._kind(x)
        rr = [int(r) % self.slot_count for r in rs]
        if kx != "ct" or not all(rr):
            raise TypeError("rotsum expects a ciphertext and non-zero rotations")
        self.ledger.record("Rot", steps)
        self.ledger.record("Add", steps)
        self.extra["KeySwitch"] += 1
        return RnsBlock(self, self.p.rotsum(vx.data, vx.level, [self.p.galois(r) for r in rr]), vx.level)

    def mult_sum(self, xs, ys):
        """add(...add(mult(x0, y0), mult(x1, y1))...) with one relinearisation
        and one rescale for the whole sum: the ledger records
        the n Mult and n - 1 Add of the separate ops.  Operands must be
        ciphertexts at one level >= 1; anything else takes the separate ops."""
        blocks = list(xs) + list(ys)
        if (len(xs) < 2 or not all(isinstance(b, RnsBlock) for b in blocks)
                or len({b.level for b in blocks}) != 1 or blocks[0].level < 1):
            acc = self.mult(xs[0], ys[0])
            for x, y in zip(xs[1:], ys[1:]):
                acc = self.add(acc, self.mult(x, y))
            return acc
        lv = blocks[0].level
        self.ledger.record("Mult", len(xs))
        self.ledger.record("Add", len(xs) - 1)
        self.extra["KeySwitch"] += 1
        return RnsBlock(self, self.p.mult_sum([x.data for x in xs], [y.data for y in ys], lv), lv - 1)

    def conj(self, x):
        kx, vx = self._kind(x)
        if kx != "ct":
            return S.Slots(np.conj(vx), S.PLAIN_LEVEL, False)
        self.ledger.record("Conj")
        self.extra["KeySwitch"] += 1
        return RnsBlock(self, self.p.automorph(vx.data, vx.level, 2 * self.p.N - 1), vx.level)

    def mul_i(self, x):
        kx, vx = self._kind(x)
        if kx != "ct":
            return S.Slots(vx * 1j, S.PLAIN_LEVEL, False)
        return RnsBlock(self, self.p.mul_i(vx.data, vx.level), vx.level)

    def bootstrap(self, x):
        if not isinstance(x, RnsBlock):
            return x
        self.ledger.record("Bootstrap")
        return self._refresh(x)

    def note_decode(self, role, tag=None):
        self.decode_events.append((role, tag))

    def decodes_by(self, role):
        return [e for e in self.decode_events if e[0] == role]
