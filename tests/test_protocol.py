"""Protocol format v2 (paper_2403_14111_b200/protocol.py) without a GPU:
framing, message typing and every malformed-input error of the reference's
channel (protocol.py:92-216), on plaintext-block matrices."""

import struct

import numpy as np
import pytest

from paper_2403_14111_b200 import protocol as PR
from paper_2403_14111_b200.context import PlainBlock
from paper_2403_14111_b200.encoding import EncodedMatrix
from paper_2403_14111_b200.errors import ProtocolError


class FakeCtx:
    """Geometry and modulus chain only (no device): enough for plaintext matrices."""

    def __init__(self, moduli=(17, 19, 23), slots=256, rows=16, logn=9):
        self.slot_count, self.grid_rows, self.grid_cols = slots, rows, slots // rows
        self.logN, self.moduli, self.max_level = logn, np.array(moduli, np.uint64), len(moduli) - 1


def _matrix(ctx, gr=1, gc=2, seed=0):
    rng = np.random.default_rng(seed)
    blocks = tuple(tuple(PlainBlock(rng.standard_normal(ctx.slot_count) + 1j * rng.standard_normal(ctx.slot_count))
                         for _ in range(gc)) for _ in range(gr))
    return EncodedMatrix(ctx, blocks, (10, 20), "horizontal", 16)


def test_plain_roundtrip_and_framing():
    ctx = FakeCtx()
    M = _matrix(ctx, 2, 3)
    data = PR.pack_matrix(M)
    assert data[0] == PR.MATRIX_VERSION
    R, pos = PR.unpack_matrix(ctx, data)
    assert pos == len(data) and R.shape == M.shape and R.tiling == "horizontal" and R.period == 16
    for ra, rb in zip(M.blocks, R.blocks):
        for a, b in zip(ra, rb):
            np.testing.assert_array_equal(a.slots, b.slots)
    a, b = PR.channel_pair()
    a.send_batch(M, M)
    a.send_stop_signal(PR.DECISION_IMPROVED)
    assert b.pending()
    f, l = b.recv_batch(ctx)
    assert f.grid == (2, 3) and l.grid == (2, 3)
    assert b.recv_stop_signal() == PR.DECISION_IMPROVED
    assert not b.pending()


def test_malformed_messages_raise_protocol_error():
    ctx = FakeCtx()
    data = bytearray(PR.pack_matrix(_matrix(ctx)))
    with pytest.raises(ProtocolError, match="version"):
        PR.unpack_matrix(ctx, bytes([1]) + bytes(data[1:]))
    with pytest.raises(ProtocolError, match="truncated matrix header"):
        PR.unpack_matrix(ctx, bytes(data[:10]))
    with pytest.raises(ProtocolError, match="truncated matrix body"):
        PR.unpack_matrix(ctx, bytes(data[:-5]))
    with pytest.raises(ProtocolError, match="context mismatch"):
        PR.unpack_matrix(FakeCtx(slots=512, rows=16), bytes(data))
    with pytest.raises(ProtocolError, match="modulus chain"):
        PR.unpack_matrix(FakeCtx(moduli=(17, 19, 29)), bytes(data))
    bad = bytearray(data)
    bad[1 + 4 + 4] = 7      # tiling code (after version, rows, cols)
    with pytest.raises(ProtocolError, match="tiling"):
        PR.unpack_matrix(ctx, bytes(bad))
    a, b = PR.channel_pair()
    with pytest.raises(ProtocolError, match="unknown message type"):
        a.send(9, b"")
    with pytest.raises(ProtocolError, match="invalid stop-signal"):
        a.send_stop_signal(5)
    with pytest.raises(ProtocolError, match="no message pending"):
        b.recv()
    a.send(PR.MSG_STOP, bytes([1]))
    with pytest.raises(ProtocolError, match="expected FinalWeights"):
        b.recv_weights(ctx)
    a.send(PR.MSG_STOP, bytes([9]))
    with pytest.raises(ProtocolError, match="malformed stop signal"):
        b.recv_stop_signal()
    a.send(PR.MSG_WEIGHTS, bytes(data) + b"xx")
    with pytest.raises(ProtocolError, match="stray bytes"):
        b.recv_weights(ctx)
    a._tx += struct.pack("<I", 100) + b"\x01"
    with pytest.raises(ProtocolError, match="truncated frame"):
        b.recv()


def test_plain_marker_in_encrypted_matrix_rejected():
    ctx = FakeCtx()
    data = bytearray(PR.pack_matrix(_matrix(ctx)))
    enc_flag = PR._HEAD.size - 1 - 2 - 8 - 1   # u8 encrypted sits before log2 N, moduli count, digest
    data[enc_flag] = 1
    with pytest.raises(ProtocolError, match="plaintext block marker"):
        PR.unpack_matrix(ctx, bytes(data))
