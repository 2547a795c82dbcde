"""TEST INFRASTRUCTURE -- restatement of the CKKS bootstrapping spec
 over the C oracle's exact primitives, the residue oracle for
the product's native bootstrap (csrc/bootstrap.cu).

The reference has no bootstrapping (its ``bootstrap`` is a level reset,
emulator.py:267-273; the paper used HEaaN's) and HEaaN is
not a dependency, so this restates the standard RNS-CKKS algorithm
(ModRaise, CoeffToSlot, EvalMod, SlotToCoeff) with every free choice pinned:

* ModRaise: level-0 coefficients centred mod q0, lifted to q_0..q_L.
* CoeffToSlot: the inverse of the slot map V (V_jk = zeta^(5^j k)) factors
  into log2(n) butterfly levels B_l^-1 (B_l: blocks n / 2^(l-1), twiddle
  zeta^(5^j 2^(l-1))); three groups of consecutive levels are merged, each a
  set of diagonals (offset d: (M x)_j += diag_d[j] x_(j+d)) applied by
  baby-step giant-step: babies lrot(x, b s), per giant g the raw ct x pt
  products summed, one rescale, lrot by g n1 s.  Every matrix entry is
  +-2^-r zeta^E with an exact integer exponent E; values are
  f * (cos(pi E / N), sin(pi E / N)), f folding the group's constant.
  The output holds the coefficients T, complex-packed and bit-reversed, at
  slot scale Delta_L; one scalar product by Delta_L / (2 K q0) (a uniform,
  scale-like rounding, unlike a factor folded into the diagonals, whose
  per-entry rounding against the ~2^64 raised values would be noise) gives
  u = x / (2K), x = T / q0.
* Real / imaginary split: u + conj(u), -i (u - conj(u)).
* EvalMod: Chebyshev series (degree 27) of cos(2 pi (K u - 1/4) / 2^4) in u,
  T_k by T_2a = 2 T_a^2 - 1 / T_k = 2 T_a T_b - T_(a-b) (a the largest power
  of two below k), terms c_k T_k at one level, then four double angles
  c <- 2 c^2 - 1: sin(2 pi x), whose 1/(2 pi) is folded into SlotToCoeff.
* Exact integer gain 2^15, recombination re + i im, SlotToCoeff (the three
  forward groups, innermost first) landing at the application top level.
"""

from __future__ import annotations

import math

import numpy as np

K_RANGE = 16             # |x| = |T / q0| bound (ModRaise overflow I plus the message)
DOUBLINGS = 4
INT_GAIN = 1 << 15       # exact integer gain before SlotToCoeff
CHEB = (0.21921621501751104, -0.04163425650808503, 0.5729882897213429, -0.005706988408963243,
        0.6283207584137114, 0.07308641363683221, -0.5527025194229122, -0.030879541430194817,
        0.14588477734714397, 0.005709279677339937, -0.020179274144300055, -0.0006170816570300078,
        0.0017582253584081749, 4.4379335769130696e-05, -0.0001063328757854582, -2.291335574193446e-06,
        4.746072353514685e-06, 8.935411073699164e-08, -1.6317891342227947e-07, -2.730062564463901e-09,
        4.461227928980592e-09, 6.71974137060941e-11, -9.940233410834453e-11, -1.3618179787512087e-12,
        1.840671891504253e-12, 2.3454661363066562e-14, -2.95837563102632e-14, -5.269516377095246e-16)


def groups(L: int, ng: int = 3):
    """Split butterfly levels 1..L into ng consecutive groups (earlier ones larger)."""
    base, extra = divmod(L, ng)
    out, lo = [], 1
    for g in range(ng):
        sz = base + (1 if g < extra else 0)
        out.append(list(range(lo, lo + sz)))
        lo += sz
    return out


def _merged(N: int, levels, inverse: bool):
    """Rows of the merged group: (cols, exps), each (n, 2^r) integer arrays.
    inverse: B_last^-1 ... B_first^-1 (CoeffToSlot), else B_first ... B_last."""
    n = N // 2
    j = np.arange(n, dtype=np.int64)
    cols = j[:, None].copy()
    exps = np.zeros((n, 1), np.int64)
    order = list(reversed(levels)) if inverse else list(levels)
    for lv in order:
        bs = n >> (lv - 1)
        h = bs // 2
        cin = cols % bs
        top = cin < h
        jj = np.where(top, cin, cin - h)
        E = (np.array([pow(5, int(v), 2 * N) for v in range(h)], np.int64)[jj] * (1 << (lv - 1))) % (2 * N)
        if inverse:
            # row c of B^-1: top (c, 0), (c + h, 0); bottom (c - h, -E), (c, N - E)
            c1 = np.where(top, cols, cols - h)
            c2 = np.where(top, cols + h, cols)
            e1 = np.where(top, 0, -E)
            e2 = np.where(top, 0, N - E)
        else:
            # row c of B: top (c, 0), (c + h, E); bottom (c - h, 0), (c, E + N)
            c1 = np.where(top, cols, cols - h)
            c2 = np.where(top, cols + h, cols)
            e1 = np.zeros_like(E)
            e2 = np.where(top, E, E + N)
        cols = np.concatenate([c1, c2], axis=1)
        exps = (np.concatenate([exps + e1, exps + e2], axis=1)) % (2 * N)
    return cols, exps


def zeta_table(N: int):
    re = np.array([math.cos(math.pi * e / N) for e in range(2 * N)])
    im = np.array([math.sin(math.pi * e / N) for e in range(2 * N)])
    return re, im


def group_plan(N: int, levels, inverse: bool, factor: float, tab):
    """BSGS plan of one merged group: step s, n1, {g: {b: pre-rotated diagonal}}."""
    n = N // 2
    r = len(levels)
    s = n >> levels[-1]
    cols, exps = _merged(N, levels, inverse)
    f = math.ldexp(1.0, -r) * factor if inverse else factor
    j = np.arange(n)[:, None]
    offs = (cols - j) % n
    diags = {}
    for col in range(offs.shape[1]):
        for d in np.unique(offs[:, col]):
            rows = np.nonzero(offs[:, col] == d)[0]
            v = diags.setdefault(int(d), np.zeros(n, np.complex128))
            e = exps[rows, col]
            v.real[rows] = f * tab[0][e]
            v.imag[rows] = f * tab[1][e]
    ks = {}
    for d, v in diags.items():
        k = d // s
        if k >= (n // s) // 2:
            k -= n // s
        ks[k] = v
    n1 = 1
    while n1 * n1 < len(ks):
        n1 *= 2
    plan = {}
    for k in sorted(ks):
        g, b = k // n1, k % n1
        G = (g * n1 * s) % n
        plan.setdefault(g, {})[b] = np.roll(ks[k], G)
    return s, n1, plan


class Bootstrapper:
    """Oracle bootstrap over RnsParams (the raw C primitives)."""

    def __init__(self, p, app_level: int):
        self.p, self.app = p, app_level
        self.N, self.n = p.N, p.N // 2
        self.L = p.L
        lg = int(math.log2(self.n))
        self.groups = groups(lg)
        tab = zeta_table(self.N)
        q0 = float(p.moduli[0])
        c_cts = float(p.scales[self.L]) / (2.0 * K_RANGE * q0)
        c_stc = q0 / (2.0 * math.pi * float(p.scales[0]) * INT_GAIN)
        self.c_cts = c_cts
        self.cts = [group_plan(self.N, g, True, 1.0, tab) for g in self.groups]
        inner = list(reversed(self.groups))
        self.stc = [group_plan(self.N, g, False, c_stc if i == 0 else 1.0, tab) for i, g in enumerate(inner)]

    # -- helpers on [2][l+1][N] residues -----------------------------------
    def _adj(self, a, frm, to):
        return a if frm == to else self.p.level_adjust(a, frm, to)

    def _rot(self, a, level, r):
        r %= self.n
        return a if r == 0 else self.p.automorph(a, level, self.p.galois(r))

    def linear(self, a, level, plan):
        s, n1, gplan = plan
        bs = sorted({b for g in gplan.values() for b in g})
        baby = {b: self._rot(a, level, b * s) for b in bs}
        outer = None
        for g in sorted(gplan):
            acc = None
            for b in sorted(gplan[g]):
                pt = self.p.encode_ntt(gplan[g][b], level)
                prod = self.p.mul_pt_raw(baby[b], pt, level)
                acc = prod if acc is None else self.p.add(acc, prod, level)
            inner = self._rot(self.p.rescale(acc, level), level - 1, g * n1 * s)
            outer = inner if outer is None else self.p.add(outer, inner, level - 1)
        return outer, level - 1

    def evalmod(self, u, lu):
        p = self.p
        T = {1: (u, lu)}
        D = len(CHEB) - 1
        for k in range(2, D + 1):
            a = 1 << (k.bit_length() - 1)
            b = k - a
            if b == 0:
                x, lx = T[k // 2]
                t = p.mult(x, x, lx)
                lt = lx - 1
            else:
                (x, lx), (y, ly) = T[a], T[b]
                lm = min(lx, ly)
                t = p.mult(self._adj(x, lx, lm), self._adj(y, ly, lm), lm)
                lt = lm - 1
            t = p.add(t, t, lt)
            if b == 0:
                T[k] = (p.add_const(t, lt, -1.0), lt)
            else:
                z, lz = T[a - b]
                T[k] = (p.add(t, self._adj(z, lz, lt), lt, negate=True), lt)
        lmin = min(l for _, l in T.values())
        acc = None
        for k in range(1, D + 1):
            x, lx = T[k]
            term = p.mul_const(self._adj(x, lx, lmin), lmin, CHEB[k])
            acc = term if acc is None else p.add(acc, term, lmin - 1)
        lc = lmin - 1
        acc = p.add_const(acc, lc, CHEB[0])
        for _ in range(DOUBLINGS):
            t = p.mult(acc, acc, lc)
            lc -= 1
            t = p.add(t, t, lc)
            acc = p.add_const(t, lc, -1.0)
        return acc, lc

    def bootstrap(self, ct, level):
        p = self.p
        a = self._adj(ct, level, 0)
        x = p.mod_raise(a, self.L)
        lv = self.L
        for plan in self.cts:
            x, lv = self.linear(x, lv, plan)
        x = p.mul_const(x, lv, self.c_cts)
        lv -= 1
        cj = self._rot_conj(x, lv)
        ure = p.add(x, cj, lv)
        uim = p.mul_i(p.add(cj, x, lv, negate=True), lv)
        sre, ls = self.evalmod(ure, lv)
        sim, _ = self.evalmod(uim, lv)
        y = p.add(p.mul_int(sre, ls, INT_GAIN), p.mul_i(p.mul_int(sim, ls, INT_GAIN), ls), ls)
        for plan in self.stc:
            y, ls = self.linear(y, ls, plan)
        if ls != self.app:
            raise RuntimeError(f"bootstrap landed at level {ls}, expected {self.app}")
        return y

    def _rot_conj(self, a, level):
        return self.p.automorph(a, level, 2 * self.N - 1)
