"""Error classes with the reference's machine codes (hefit/errors.py:8-59)."""


class HefitError(Exception):
    code = "hefit.error"


class DepthExhausted(HefitError):
    code = "emulator.depth"


class SlotCountMismatch(HefitError):
    code = "emulator.slots"


class ShapeMismatch(HefitError):
    code = "encoding.shape"


class TilingError(HefitError):
    code = "encoding.tiling"


class ResidualImaginary(HefitError):
    code = "encoding.imaginary"
