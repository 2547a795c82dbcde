"""CKKS bootstrapping on the GPU against the oracle's
restatement (oracle/boot.py): bit-exact residues at a 2^10 ring, precision
at N = 2^16, and the reference's hot path (softmax, NAG step) with real
bootstrapping in place of the refresh surrogate -- no secret key on the
server side of the computation."""

import numpy as np
import pytest

from oracle import boot as B
from oracle import rns as R
from oracle import slots as S

pytestmark = pytest.mark.gpu

OPS = S.OP_KINDS


def _prod():
    import paper_2403_14111_b200 as P
    return P


@pytest.mark.parametrize("level", [0, 3, 12])
def test_bootstrap_residues_boot10(level):
    P = _prod()
    g = P.CKKSContext("boot10", 16, seed=5)
    o = R.RnsParams("boot10", seed=5)
    o.set_app_level(12)
    bt = B.Bootstrapper(o, 12)
    rng = np.random.default_rng(level)
    w = rng.uniform(-1, 1, g.slot_count) + 1j * rng.uniform(-1, 1, g.slot_count)
    g.nonce = 7
    x = g.encrypt(w, level)
    ox = o.encrypt(w, level, 7)
    np.testing.assert_array_equal(x.residues(), ox)
    y = g.ckks_bootstrap(x)
    oy = bt.bootstrap(ox, level)
    assert y.level == 12
    np.testing.assert_array_equal(y.residues(), oy)
    assert np.max(np.abs(y.slots - w)) < 1e-4


@pytest.mark.slow
def test_bootstrap_precision_boot16():
    """N = 2^16 (2^15 slots): the refreshed message within 1e-3 of the input
    over uniform complex slots in the unit box and over large real values
    (the softmax refreshes values up to ~2^7)."""
    P = _prod()
    g = P.CKKSContext("boot16", 128, seed=5)
    rng = np.random.default_rng(1)
    for scale in (1.0, 100.0):
        w = scale * (rng.uniform(-1, 1, g.slot_count) + (1j if scale == 1.0 else 0) * rng.uniform(-1, 1, g.slot_count))
        x = g.encrypt(w, 0)
        y = g.ckks_bootstrap(x)
        assert y.level == g.max_level == 12
        err = np.max(np.abs(y.slots - w))
        assert err < 1e-3 * max(1.0, scale / 10), (scale, err)


def test_softmax_with_ckks_bootstrapping_boot10(golden):
    """The reference's softmax with every auto-bootstrap a real CKKS
    bootstrapping: residues and ledger equal the oracle's restated run, values
    within 1e-2 of the reference emulator's (a 16 x 32 grid here)."""
    P = _prod()
    g = P.CKKSContext("boot10", 16, seed=8, auto_bootstrap=True, bootstrap="ckks")
    o = R.OracleCKKSContext("boot10", 16, seed=8, auto_bootstrap=True, bootstrap="ckks")
    Z = golden["small_sm_in"]
    g.nonce = o.nonce = 0
    GM, OM = P.encode(g, Z, "horizontal"), S.encode(o, Z, "horizontal")
    out = P.a_softmax(GM)
    ref = S.a_softmax(OM)
    for bg, bo in zip(out.flat(), [b for r in ref.blocks for b in r]):
        np.testing.assert_array_equal(bg.residues(), bo.data)
    assert g.nonce == o.nonce
    led = g.ledger.counts()
    assert [led[k] for k in OPS] == [o.ledger.counts()[k] for k in OPS]
    assert led["Bootstrap"] > 0
    assert np.max(np.abs(P.decode(out, tol=1e-2) - golden["small_sm_out"])) < 1e-2


@pytest.mark.slow
def test_config4_step_with_ckks_bootstrapping(golden):
    """BASELINE config 4, first 128-row NAG step at N = 2^16 with real CKKS
    bootstrapping (54 per step) instead of the secret-key refresh: the
    reference's ledger and the weights against the reference's snapshot."""
    P = _prod()
    from paper_2403_14111_b200 import workloads as wl
    X, y = wl.config4()
    Y = P.one_hot(y, wl.CLASSES)
    g = P.CKKSContext("boot16", 128, seed=4, auto_bootstrap=True, bootstrap="ckks")
    w0 = P.init_weights(wl.CLASSES, X.shape[1], wl.INIT_SEED)
    W = P.encode(g, w0, "vertical")
    st = P.TrainState(W, W)
    P.nag_step(st, P.encode(g, X[:128]), P.encode(g, Y[:128], "horizontal"), wl.LEARNING_RATE, 128)
    led = g.ledger.counts()
    assert [led[k] for k in OPS] == [518, 101, 164, 382, 4, 54]
    w1 = P.decode(st.weights, tol=1e-2)
    assert np.max(np.abs(w1 - golden["cfg4_snaps"][0])) < 2e-3


@pytest.mark.slow
@pytest.mark.parametrize("level", [29, 20])
def test_keyswitch_eight_digits_boot16(level):
    """The fused key switch with 8 digits (the bootstrapping chain's upper
    levels, dnum > 4): rotation, conjugation and relinearised product
    residues equal the oracle's at N = 2^16."""
    P = _prod()
    g = P.CKKSContext("boot16", 128, seed=9)
    o = R.OracleCKKSContext("boot16", 128, seed=9)
    rng = np.random.default_rng(level)
    x = rng.uniform(-1, 1, g.slot_count) + 1j * rng.uniform(-1, 1, g.slot_count)
    p = o.p   # raw oracle primitives: levels above the application's
    ox = p.encrypt(x, level, 3)
    gx = g.from_residues(ox, level)
    np.testing.assert_array_equal(g.lrot(gx, 5).residues(), p.automorph(ox, level, p.galois(5)))
    np.testing.assert_array_equal(g.conj(gx).residues(), p.automorph(ox, level, 2 * p.N - 1))
    np.testing.assert_array_equal(g.mult(gx, gx).residues(), p.mult(ox, ox, level))
