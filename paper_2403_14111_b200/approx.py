"""Approximate softmax on the B200 backend (API of hefit.approx, approx.py:38-344).

``a_softmax`` on an encrypted, horizontally tiled, single-block-column matrix
runs as one native schedule (csrc/schedules.cu) with the reference's op
order: tournament max (log2(period) rounds of f∘g∘g comparisons), domain
extension, degree-5 compensation, degree-12 exp + squarings, col_sums and
16 Goldschmidt iterations, with the refresh surrogate at every level-0
multiplication operand exactly where the reference auto-bootstraps.
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
