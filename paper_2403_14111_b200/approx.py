"""Approximate softmax on the B200 backend (API of hefit.approx, approx.py:38-344).

``a_softmax`` on an encrypted, horizontally tiled, single-block-column matrix
runs as one native schedule (csrc/schedules.cu) with the reference's op
order: tournament max (log2(period) rounds of f∘g∘g comparisons), domain
extension, degree-5 compensation, degree-12 exp + squarings, col_sums and
16 Goldschmidt iterations, with the refresh surrogate at every level-0
multiplication operand exactly where the reference auto-bootstraps.
The building blocks ``a_comp`` / ``a_max`` / ``domain_extend`` / ``a_exp`` /
``a_inv`` (hefit/__init__.py:22-28) are exported the same way, each one
native call (``hc_approx``) over all blocks of its operand in lockstep.
The float64 array carrier of the reference is its plaintext twin; it lives in
the test oracle (oracle/slots.py), not in this package.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

from . import _native as N
from .context import Ciphertext
from .encoding import EncodedMatrix
from .errors import ShapeMismatch
from .matmul import _handles, _native_ctx

# frozen constants (hefit/_constants.py:7-21, approx.py:34-35)
EXP_POLY = (
    0.9999999999999948, 0.9999999999996788, 0.5000000000004744, 0.1666666666766445,
    0.04166666666019774, 0.00833333324592319, 0.0013888889188354027, 0.00019841302319140728,
    2.4801530417934142e-05, 2.7551504280360845e-06, 2.7561173628426655e-07, 2.5547752396936175e-08,
    2.0934824859870782e-09,
)
COMP_F = (35 / 16, -35 / 16, 21 / 16, -5 / 16)
COMP_G = (4589 / 1024, -16577 / 1024, 25614 / 1024, -12860 / 1024)


@dataclass(frozen=True)
class SoftmaxConfig:
    base_range: float = 8.0
    extension_base: float = 2.0
    extension_steps: int = 5
    precise: bool = True
    exp_range: int = 8
    inv_range: float = 100.0
    inv_iters: int = 16

    @property
    def max_range(self) -> int:
        return int(math.ceil(self.base_range * self.extension_base ** self.extension_steps / 2))

    @property
    def dep_delta(self) -> float:
        return 4.0 / (27.0 * self.base_range ** 2)

    def as_array(self):
        return (C.c_double * 7)(self.base_range, self.extension_base, float(self.extension_steps),
                                1.0 if self.precise else 0.0, float(self.exp_range), self.inv_range,
                                float(self.inv_iters))


DEFAULTS = SoftmaxConfig()


def a_softmax(M: EncodedMatrix, cfg: SoftmaxConfig = DEFAULTS, classes: int | None = None,
              period: int | None = None) -> EncodedMatrix:
    """Row-wise approximate softmax of encrypted logits (approx.py:312-344).

    Needs ``ctx.auto_bootstrap = True`` at realistic depths, as in the reference."""
    if not isinstance(M, EncodedMatrix):
        raise TypeError("a_softmax on the B200 backend takes an encrypted EncodedMatrix "
                        "(the float64 array carrier is the plaintext twin, see oracle/slots.py)")
    if M.tiling != "horizontal" or M.grid[1] != 1:
        raise ShapeMismatch("softmax expects a horizontally tiled single-block-column matrix")
    ctx = _native_ctx(M)
    classes = M.shape[1] if classes is None else classes
    period = M.period if period is None else period
    if period < classes:
        raise ShapeMismatch(f"period {period} smaller than classes {classes}")
    m = M.grid[0]
    out = (C.c_void_p * m)()
    counts = (C.c_int64 * N.NCOUNTS)()
    N.check(N.lib().hc_softmax(ctx._h, _handles(M.flat()), m, classes, period, cfg.as_array(), out, counts))
    blocks = tuple((Ciphertext(ctx, C.c_void_p(out[p])),) for p in range(m))
    return EncodedMatrix(ctx, blocks, (M.shape[0], classes), "horizontal", period)


# -- building blocks (approx.py:195-309), encrypted carrier ----------------------

HC_APPROX_COMP, HC_APPROX_MAX, HC_APPROX_DOMAIN_EXTEND, HC_APPROX_DEP_COMP, HC_APPROX_EXP, HC_APPROX_INV = range(6)


def _approx(fn: int, M: EncodedMatrix, cfg: SoftmaxConfig, other: EncodedMatrix | None = None, classes: int = 0,
            period: int = 0) -> EncodedMatrix:
    if not isinstance(M, EncodedMatrix):
        raise TypeError("the B200 backend takes an encrypted EncodedMatrix "
                        "(the float64 array carrier is the plaintext twin, see oracle/slots.py)")
    ctx = _native_ctx(M) if other is None else _native_ctx(M, other)
    if other is not None and (other.grid != M.grid):
        raise ShapeMismatch(f"operand grids differ: {M.grid} vs {other.grid}")
    blocks = M.flat()
    out = (C.c_void_p * len(blocks))()
    counts = (C.c_int64 * N.NCOUNTS)()
    N.check(N.lib().hc_approx(ctx._h, fn, _handles(blocks), _handles(other.flat()) if other is not None else None,
                              len(blocks), classes, period, cfg.as_array(), out, counts))
    m, n = M.grid
    res = tuple(tuple(Ciphertext(ctx, C.c_void_p(out[p * n + q])) for q in range(n)) for p in range(m))
    return EncodedMatrix(ctx, res, M.shape, M.tiling, M.period)


def a_comp(x: EncodedMatrix, y: EncodedMatrix) -> EncodedMatrix:
    """Soft comparison (approx.py:205-213): ~1 where x > y, 1/2 at equality;
    f o g o g of odd degree-7 polynomials on inputs in [-1/2, 1/2]."""
    return _approx(HC_APPROX_COMP, x, DEFAULTS, other=y)


def a_max(M: EncodedMatrix, cfg: SoftmaxConfig = DEFAULTS, classes: int | None = None,
          period: int | None = None) -> EncodedMatrix:
    """Row-wise approximate maximum broadcast over the row (approx.py:216-238)."""
    if M.tiling != "horizontal" or M.grid[1] != 1:
        raise ShapeMismatch("a_max expects a horizontally tiled single-block-column matrix")
    classes = M.shape[1] if classes is None else classes
    period = M.period if period is None else period
    if period < classes:
        raise ShapeMismatch(f"period {period} smaller than classes {classes}")
    return _approx(HC_APPROX_MAX, M, cfg, classes=classes, period=period)


def domain_extend(M: EncodedMatrix, cfg: SoftmaxConfig = DEFAULTS) -> EncodedMatrix:
    """Contract [-max_range, max_range] into the exp's base range (approx.py:241-253)."""
    return _approx(HC_APPROX_DOMAIN_EXTEND, M, cfg)


def dep_compensation(M: EncodedMatrix, cfg: SoftmaxConfig = DEFAULTS) -> EncodedMatrix:
    """Degree-5 correction of the contraction bias (approx.py:256-273, ``_dep_compensation``)."""
    return _approx(HC_APPROX_DEP_COMP, M, cfg)


def a_exp(M: EncodedMatrix, cfg: SoftmaxConfig = DEFAULTS) -> EncodedMatrix:
    """exp on [-exp_range, exp_range]: degree-12 fit at x/B, squared log2(B) times (approx.py:276-292)."""
    if cfg.exp_range < 1 or cfg.exp_range & (cfg.exp_range - 1):
        raise ShapeMismatch(f"exp_range must be a power of two, got {cfg.exp_range}")
    return _approx(HC_APPROX_EXP, M, cfg)


def a_inv(M: EncodedMatrix, cfg: SoftmaxConfig = DEFAULTS) -> EncodedMatrix:
    """Goldschmidt reciprocal normalised by inv_range (approx.py:295-309)."""
    return _approx(HC_APPROX_INV, M, cfg)

