"""B200-native RNS-CKKS backend for the HETAL hot path (arXiv 2403.14111).

Drop-in for the reference package's hot path (``hefit``): the backend
interface (``CKKSContext`` ~ ``EmulatorContext``), matrix encoding and the
structural ops, DiagABT / DiagATB, the approximate softmax and the NAG
training step — with ciphertexts resident in B200 HBM and every op a
hand-written sm_100a CUDA kernel sequence behind the C-ABI in include/hc.h.
"""

from .approx import (
    COMP_F,
    COMP_G,
    DEFAULTS,
    EXP_POLY,
    SoftmaxConfig,
    a_comp,
    a_exp,
    a_inv,
    a_max,
    a_softmax,
    dep_compensation,
    domain_extend,
)
from .context import (
    DECODE_TOL,
    DEFAULT_OP_WEIGHTS_MS,
    OP_KINDS,
    PARAMS,
    Ciphertext,
    CKKSContext,
    NativeLedger,
    PlainBlock,
)
from .encoding import (
    EncodedMatrix,
    col_range_mask,
    col_sums,
    decode,
    encode,
    make_mask,
    next_pow2,
    padded_array,
    pattern_matrix,
    prot_up,
    rot_left,
    rot_up,
    row_sums,
)
from .errors import (
    DepthExhausted,
    HefitError,
    ProtocolError,
    ResidualImaginary,
    ShapeMismatch,
    SlotCountMismatch,
    TilingError,
)
from .matmul import ALGORITHMS, col_major_abt, count_formula, diag_abt, diag_atb, rotation_steps, row_major_atb
from .protocol import ChannelEndpoint, channel_pair, pack_matrix, unpack_matrix
from .training import (
    Client,
    FitResult,
    Server,
    TrainState,
    batch_slices,
    fit,
    init_weights,
    log_loss,
    nag_step,
    one_hot,
    default_context,
    run_steps,
)

__version__ = "0.1.0"
