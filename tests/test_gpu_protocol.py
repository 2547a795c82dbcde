"""GPU: protocol format v2 carries device ciphertexts bit-exactly, and the
two-party ``fit`` (validation logits, early stopping, final weights) on
RNS-CKKS reproduces the reference's own run (golden vectors from
training.fit, tests/golden/make_golden.py) — same decisions and ledger,
values within CKKS tolerance."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

OPS = ("Add", "CMult", "Mult", "Rot", "Conj", "Bootstrap")


def test_ciphertext_roundtrip_bit_exact():
    import paper_2403_14111_b200 as P
    from paper_2403_14111_b200 import protocol as PR
    g = P.CKKSContext("small12", 16, seed=21)
    rng = np.random.default_rng(0)
    X = rng.uniform(-1, 1, (16, 40))
    E = P.encode(g, X)
    low = E.blocks[0][1]
    E2 = P.EncodedMatrix(g, ((E.blocks[0][0], g.mult(low, low), E.blocks[0][2]),), E.shape, E.tiling, E.period)
    data = PR.pack_matrix(E2)
    R, pos = PR.unpack_matrix(g, data)
    assert pos == len(data) and R.grid == E2.grid
    for a, b in zip(E2.flat(), R.flat()):
        assert a.level == b.level
        np.testing.assert_array_equal(a.residues(), b.residues())
    np.testing.assert_allclose(P.decode(R)[:, :16], X[:, :16], atol=1e-5)
    # a residue at or above its modulus is rejected
    bad = bytearray(data)
    off = PR._HEAD.size + PR._LEVEL.size
    bad[off:off + 8] = int(g.moduli[0]).to_bytes(8, "little")
    with pytest.raises(P.ProtocolError, match="out of range"):
        PR.unpack_matrix(g, bytes(bad))
    # a receiver on another ring / chain is rejected
    with pytest.raises(P.ProtocolError, match="context mismatch"):
        PR.unpack_matrix(P.CKKSContext("tiny", 16, seed=21), data)


def test_fit_matches_reference_run(golden):
    import paper_2403_14111_b200 as P
    g = P.CKKSContext("small12", 16, seed=31, auto_bootstrap=True)
    r = P.fit(golden["fit_xt"], golden["fit_yt"], golden["fit_xv"], golden["fit_yv"], 3, ctx=g, lr=1.0,
              batch_size=16, epochs=8, patience=2, seed=1)
    meta = golden["fit_meta"]
    assert [r.epochs_run, r.best_epoch, int(r.stopped_early)] == list(meta)
    assert [r.ledger_counts[k] for k in OPS] == list(golden["fit_led"])
    np.testing.assert_allclose(r.val_losses, golden["fit_val_losses"], atol=1e-3)
    np.testing.assert_allclose(r.train_losses, golden["fit_train_losses"], atol=1e-3)
    np.testing.assert_allclose(r.weights, golden["fit_weights"], atol=1e-3)
    assert g.decodes_by("server") == []
    assert len(g.decodes_by("client")) == r.epochs_run + 1


def test_async_transfers_match_sync_path():
    """hc_ct_upload_async / hc_ct_download_async (copy streams) give the
    residues of the synchronous path, with work issued in between."""
    import ctypes as C

    import paper_2403_14111_b200 as P
    from paper_2403_14111_b200 import _native as N
    g = P.CKKSContext("small12", 16, seed=41)
    rng = np.random.default_rng(2)
    x = rng.uniform(-1, 1, g.slot_count)
    ct = g.encrypt(x)
    res = np.ascontiguousarray(ct.residues())
    L = N.lib()
    h = C.c_void_p()
    N.check(L.hc_ct_upload_async(g._h, res.ctypes.data_as(N.U64P), ct.level, C.byref(h)))
    up = P.Ciphertext(g, h)
    sq = g.mult(up, up)
    out = np.zeros((2, sq.level + 1, g.N), np.uint64)
    N.check(L.hc_ct_download_async(sq._h, out.ctypes.data_as(N.U64P)))
    ref = g.mult(ct, ct)
    g.sync()
    np.testing.assert_array_equal(out, ref.residues())
    np.testing.assert_array_equal(up.residues(), res)
