"""The bench's roofline numerator: SURVEY §8(d)'s per-op HBM model, which the
library accumulates op by op (hc_ctx_model_bytes), must equal the same model
traced over the unmodified reference running the same computation.

The trace wraps hefit's EmulatorContext and charges every ledgered op at its
level (Add 6/5/4 Lq, CMult 5Lq-2 / 4Lq-2, Mult 4Lq + 2d(Lq+K) + 2(Lq-1),
Rot/Conj 4Lq + 2d(Lq+K), MulI 4Lq limbs of 8N bytes; Lq = active primes of the
operation's input).  SURVEY §8(d) quotes 19.98 GB (DiagABT cfg1) and
21.21 GB (DiagATB-RL cfg2)."""

import math

import numpy as np
import pytest

N16, K, ALPHA = 1 << 16, 3, 4


def _limbs(kind, variant, level):
    Lq = level + 1
    d = math.ceil(Lq / ALPHA)
    if kind == "Add":
        return {"ct": 6, "pt": 5, "scalar": 4}[variant] * Lq
    if kind == "CMult":
        return (5 if variant == "pt" else 4) * Lq - 2
    if kind == "MulI":
        return 4 * Lq
    if kind == "Mult":
        return 4 * Lq + 2 * d * (Lq + K) + 2 * (Lq - 1)
    return 4 * Lq + 2 * d * (Lq + K)


def _tracing_context(hefit):
    class Trace(hefit.EmulatorContext):
        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            self.model = 0.0

        def _variant(self, v):
            if isinstance(v, hefit.CipherBlock):
                return "ct" if v.encrypted else "pt"
            if isinstance(v, (int, float, complex, np.number)):
                return "scalar"
            return "pt"

        def _charge(self, kind, variant, level):
            self.model += _limbs(kind, variant, level) * 8.0 * N16

        def add(self, x, y):
            r = super().add(x, y)
            if r.encrypted:
                vx, vy = self._variant(x), self._variant(y)
                v = "ct" if vx == vy == "ct" else ("scalar" if "scalar" in (vx, vy) else "pt")
                self._charge("Add", v, r.level)
            return r

        def sub(self, x, y):
            r = super().sub(x, y)
            if r.encrypted:
                vx, vy = self._variant(x), self._variant(y)
                v = "ct" if vx == vy == "ct" else ("scalar" if "scalar" in (vx, vy) else "pt")
                self._charge("Add", v, r.level)
            return r

        def mult(self, x, y):
            r = super().mult(x, y)
            vx, vy = self._variant(x), self._variant(y)
            if vx == vy == "ct":
                self._charge("Mult", "ct", r.level + 1)
            elif "ct" in (vx, vy):
                self._charge("CMult", "scalar" if "scalar" in (vx, vy) else "pt", r.level + 1)
            return r

        def lrot(self, x, r):
            out = super().lrot(x, r)
            if out is not x and x.encrypted:
                self._charge("Rot", "ct", x.level)
            return out

        def mul_i(self, x):
            out = super().mul_i(x)
            if x.encrypted:
                self._charge("MulI", "ct", x.level)
            return out

        def conj(self, x):
            out = super().conj(x)
            if x.encrypted:
                self._charge("Conj", "ct", x.level)
            return out

    return Trace


@pytest.mark.gpu
@pytest.mark.slow
def test_model_bytes_match_reference_trace(hefit):
    import paper_2403_14111_b200 as P
    from paper_2403_14111_b200 import workloads as wl
    Trace = _tracing_context(hefit)
    X, W = wl.config1()
    PY, _ = wl.config2()
    e = Trace(32768, 128, max_level=12)
    hefit.diag_abt(hefit.encode(e, X), hefit.encode(e, W, "vertical"))
    abt = e.model
    e.model = 0.0
    hefit.diag_atb(hefit.encode(e, PY, "horizontal"), hefit.encode(e, X))
    atb = e.model
    assert abs(abt / 1e9 - 19.98) < 0.005 and abs(atb / 1e9 - 21.21) < 0.005
    g = P.CKKSContext("cfg1", 128, seed=1)
    EX, EW, EP = P.encode(g, X), P.encode(g, W, "vertical"), P.encode(g, PY, "horizontal")
    g.model_bytes(reset=True)
    P.diag_abt(EX, EW)
    assert g.model_bytes(reset=True) == pytest.approx(abt, rel=1e-12)
    P.diag_atb(EP, EX)
    assert g.model_bytes(reset=True) == pytest.approx(atb, rel=1e-12)
