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


class ProtocolError(HefitError):
    """A channel message could not be parsed or arrived out of order (errors.py:56-59)."""

    code = "protocol.message"
