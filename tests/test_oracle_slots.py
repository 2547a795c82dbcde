"""Pin the slot-level oracle restatement (oracle/slots.py) against golden
vectors produced by the reference itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from oracle import slots as S
from paper_2403_14111_b200 import workloads as wl

OPS = S.OP_KINDS


def led(d):
    return np.array([d[k] for k in OPS])


def test_small_diag_abt(golden):
    ctx = S.SlotBackend(256, 16, max_level=12)
    b0 = ctx.ledger.snapshot()
    r = S.diag_abt(S.encode(ctx, golden["small_abt_A"]),
                   S.encode(ctx, golden["small_abt_B"], "vertical"), scale=0.25)
    np.testing.assert_array_equal(S.decode(r), golden["small_abt_out"])
    np.testing.assert_array_equal(led(ctx.ledger.delta(b0)), golden["small_abt_led"])
    assert r.level == golden["small_abt_level"]


@pytest.mark.parametrize("branch,alev", [("rl", None), ("pru", 11)])
def test_small_diag_atb(golden, branch, alev):
    ctx = S.SlotBackend(256, 16, max_level=12)
    r = S.diag_atb(S.encode(ctx, golden["small_atb_A"], "horizontal", level=alev),
                   S.encode(ctx, golden["small_atb_B"]), scale=2.0)
    np.testing.assert_array_equal(S.decode(r), golden[f"small_atb_{branch}_out"])
    np.testing.assert_array_equal(led(ctx.ledger.counts()), golden[f"small_atb_{branch}_led"])
    assert r.level == golden[f"small_atb_{branch}_level"]


def test_small_softmax(golden):
    ctx = S.SlotBackend(256, 16, max_level=12, auto_bootstrap=True)
    r = S.a_softmax(S.encode(ctx, golden["small_sm_in"], "horizontal"))
    np.testing.assert_array_equal(S.decode(r), golden["small_sm_out"])
    np.testing.assert_array_equal(led(ctx.ledger.counts()), golden["small_sm_led"])
    assert r.level == golden["small_sm_level"]


def test_array_carrier_pins(golden):
    cfg = S.SMCfg()
    np.testing.assert_array_equal(S.a_softmax(golden["arr_sm_in"], cfg), golden["arr_sm_out"])
    np.testing.assert_array_equal(S.a_max(golden["arr_sm_in"], cfg), golden["arr_max_out"])
    np.testing.assert_array_equal(S.a_exp(np.linspace(-8, 0, 101)[None, :], cfg), golden["arr_exp_out"])
    np.testing.assert_array_equal(S.a_inv(np.linspace(0.5, 150, 101)[None, :], cfg), golden["arr_inv_out"])
    c = golden["pin_comp"]
    assert S.a_comp(np.array([0.4]), np.array([-0.4]))[0] == c[0]
    assert S.a_comp(np.array([0.3]), np.array([0.3]))[0] == 0.5 == c[1]


def test_small_training_steps(golden):
    x, y = golden["small_train_x"], golden["small_train_y"]
    ctx = S.SlotBackend(256, 16, max_level=12, auto_bootstrap=True)
    w0 = S.init_weights(3, x.shape[1], 7)
    W = S.encode(ctx, w0, "vertical")
    st = S.State(W, W)
    Y = S.one_hot(y, 3)
    snaps = []
    for step in range(3):
        sl = slice((step % 2) * 16, (step % 2) * 16 + 16)
        S.nag_step(st, S.encode(ctx, x[sl]), S.encode(ctx, Y[sl], "horizontal"), 0.3, 16)
        snaps.append(S.decode(st.weights))
    np.testing.assert_array_equal(np.stack(snaps), golden["small_train_snaps"])
    np.testing.assert_array_equal(led(ctx.ledger.counts()), golden["small_train_led"])


def test_config0_and_1(golden):
    A, B = wl.config0()
    ctx = S.SlotBackend(4096, 64, max_level=4)
    r = S.diag_abt(S.encode(ctx, A), S.encode(ctx, B, "vertical"))
    np.testing.assert_array_equal(S.decode(r), golden["cfg0_out"])
    np.testing.assert_array_equal(led(ctx.ledger.counts()), golden["cfg0_led"])
    np.testing.assert_allclose(S.decode(r), A @ B.T, atol=1e-12)
    X, W = wl.config1()
    ctx = S.SlotBackend(32768, 128, max_level=12)
    r = S.diag_abt(S.encode(ctx, X), S.encode(ctx, W, "vertical"))
    np.testing.assert_array_equal(S.decode(r), golden["cfg1_out"])
    np.testing.assert_array_equal(led(ctx.ledger.counts()), golden["cfg1_led"])
    assert r.level == 9


@pytest.mark.parametrize("branch,alev", [("rl", None), ("pru", 11)])
def test_config2(golden, branch, alev):
    PY, X = wl.config2()
    ctx = S.SlotBackend(32768, 128, max_level=12)
    r = S.diag_atb(S.encode(ctx, PY, "horizontal", level=alev), S.encode(ctx, X))
    np.testing.assert_array_equal(S.decode(r), golden[f"cfg2_{branch}_out"])
    np.testing.assert_array_equal(led(ctx.ledger.counts()), golden[f"cfg2_{branch}_led"])
    f = S.count_formula("diag_atb_" + branch, (128, 768, 16), 128, 256)
    assert {k: ctx.ledger.counts()[k] for k in f} == f


def test_config3(golden):
    Z = wl.config3()
    ctx = S.SlotBackend(32768, 128, max_level=12, auto_bootstrap=True)
    r = S.a_softmax(S.encode(ctx, Z, "horizontal"))
    np.testing.assert_array_equal(S.decode(r), golden["cfg3_out"])
    np.testing.assert_array_equal(led(ctx.ledger.counts()), golden["cfg3_led"])
    assert np.max(np.abs(S.decode(r) - S.exact_softmax(Z))) < 0.0097   # Table 5 c=10 bound


def test_config4_epoch(golden):
    X, y = wl.config4()
    Y = S.one_hot(y, wl.CLASSES)
    ctx = S.SlotBackend(32768, 128, max_level=12, auto_bootstrap=True)
    W = S.encode(ctx, S.init_weights(wl.CLASSES, X.shape[1], wl.INIT_SEED), "vertical")
    st = S.State(W, W)
    snaps = []
    for step in range(8):
        sl = slice(step * 128, step * 128 + 128)
        S.nag_step(st, S.encode(ctx, X[sl]), S.encode(ctx, Y[sl], "horizontal"), wl.LEARNING_RATE, 128)
        snaps.append(S.decode(st.weights))
    np.testing.assert_array_equal(np.stack(snaps), golden["cfg4_snaps"])
    np.testing.assert_array_equal(led(ctx.ledger.counts()), golden["cfg4_led"])


def test_table4_baselines(golden):
    """col_major_abt / row_major_atb (matmul.py:160-237) vs the reference."""
    ctx = S.SlotBackend(256, 16, max_level=12)
    b0 = ctx.ledger.snapshot()
    r = S.col_major_abt(S.encode(ctx, golden["small_cm_A"]), S.encode(ctx, golden["small_cm_B"]), scale=-1.0)
    np.testing.assert_array_equal(S.decode(r), golden["small_cm_out"])
    np.testing.assert_array_equal(led(ctx.ledger.delta(b0)), golden["small_cm_led"])
    assert r.level == golden["small_cm_level"]
    b0 = ctx.ledger.snapshot()
    r = S.row_major_atb(S.encode(ctx, golden["small_rm_A"]), S.encode(ctx, golden["small_rm_B"]), scale=0.5)
    np.testing.assert_array_equal(S.decode(r), golden["small_rm_out"])
    np.testing.assert_array_equal(led(ctx.ledger.delta(b0)), golden["small_rm_led"])
    assert r.level == golden["small_rm_level"]
    d = ctx.ledger.delta(b0)
    f = S.count_formula("row_major", (40, 21, 6), 16, 16)
    assert {k: d[k] for k in f} == f
