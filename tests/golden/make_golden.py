"""Generate golden vectors by running the REFERENCE itself (hefit, pure Python).

Run in the build container only (it reads /root/reference):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

Writes tests/golden/hefit_golden.npz.  The committed fixture pins
oracle/slots.py (the slot-level restatement) bit-for-bit, and gives ledger
known-answer tests for every BASELINE config.  Nothing on the GPU box reads
/root/reference; it reads this .npz instead.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

import hefit  # noqa: E402
from hefit import approx, encoding, matmul, training  # noqa: E402
from hefit.emulator import EmulatorContext  # noqa: E402

from paper_2403_14111_b200 import workloads as wl  # noqa: E402

OPS = ("Add", "CMult", "Mult", "Rot", "Conj", "Bootstrap")


def led(d):
    return np.array([d[k] for k in OPS], dtype=np.int64)


def main():
    out = {}
    rng = np.random.default_rng(12345)

    # -- small grid (tests/conftest.py:8-11 geometry: 256 slots, 16x16) -----
    ctx = EmulatorContext(256, 16, max_level=12)
    A = rng.uniform(-1, 1, (10, 16))
    B = rng.uniform(-1, 1, (4, 16))
    out["small_abt_A"], out["small_abt_B"] = A, B
    b0 = ctx.ledger.snapshot()
    r = matmul.diag_abt(encoding.encode(ctx, A), encoding.encode(ctx, B, "vertical"), scale=0.25)
    out["small_abt_out"] = encoding.decode(r)
    out["small_abt_led"] = led(ctx.ledger.delta(b0))
    out["small_abt_level"] = np.array(r.level)

    At = rng.uniform(-1, 1, (16, 4))
    Bt = rng.uniform(-1, 1, (16, 21))
    out["small_atb_A"], out["small_atb_B"] = At, Bt
    for name, alev in (("rl", None), ("pru", 11)):
        b0 = ctx.ledger.snapshot()
        r = matmul.diag_atb(encoding.encode(ctx, At, "horizontal", level=alev),
                            encoding.encode(ctx, Bt), scale=2.0)
        out[f"small_atb_{name}_out"] = encoding.decode(r)
        out[f"small_atb_{name}_led"] = led(ctx.ledger.delta(b0))
        out[f"small_atb_{name}_level"] = np.array(r.level)

    # Table-4 baselines (matmul.py:160-237)
    Ac = rng.uniform(-1, 1, (20, 40))
    Bc = rng.uniform(-1, 1, (5, 40))
    out["small_cm_A"], out["small_cm_B"] = Ac, Bc
    b0 = ctx.ledger.snapshot()
    r = matmul.col_major_abt(encoding.encode(ctx, Ac), encoding.encode(ctx, Bc), scale=-1.0)
    out["small_cm_out"] = encoding.decode(r)
    out["small_cm_led"] = led(ctx.ledger.delta(b0))
    out["small_cm_level"] = np.array(r.level)
    Ar = rng.uniform(-1, 1, (40, 6))
    Br = rng.uniform(-1, 1, (40, 21))
    out["small_rm_A"], out["small_rm_B"] = Ar, Br
    b0 = ctx.ledger.snapshot()
    r = matmul.row_major_atb(encoding.encode(ctx, Ar), encoding.encode(ctx, Br), scale=0.5)
    out["small_rm_out"] = encoding.decode(r)
    out["small_rm_led"] = led(ctx.ledger.delta(b0))
    out["small_rm_level"] = np.array(r.level)

    bctx = EmulatorContext(256, 16, max_level=12, auto_bootstrap=True)
    Z = rng.uniform(-100, 100, (16, 5))
    out["small_sm_in"] = Z
    b0 = bctx.ledger.snapshot()
    r = approx.a_softmax(encoding.encode(bctx, Z, "horizontal"))
    out["small_sm_out"] = encoding.decode(r)
    out["small_sm_led"] = led(bctx.ledger.delta(b0))
    out["small_sm_level"] = np.array(r.level)
    arr = rng.uniform(-128, 128, (64, 10))
    out["arr_sm_in"] = arr
    out["arr_sm_out"] = approx.a_softmax(arr)
    out["arr_max_out"] = approx.a_max(arr)
    out["pin_comp"] = np.array([approx.a_comp(np.array([0.4]), np.array([-0.4]))[0],
                                approx.a_comp(np.array([0.3]), np.array([0.3]))[0]])
    xs = np.linspace(-8, 0, 101)[None, :]
    out["arr_exp_out"] = approx.a_exp(xs)
    ys = np.linspace(0.5, 150, 101)[None, :]
    out["arr_inv_out"] = approx.a_inv(ys)

    # -- NAG steps on the small grid (training.run_steps) -------------------
    xs_ = rng.standard_normal((32, 16))
    ys_ = rng.integers(0, 3, 32)
    out["small_train_x"], out["small_train_y"] = xs_, ys_
    tctx = EmulatorContext(256, 16, max_level=12, auto_bootstrap=True)
    snaps = training.run_steps(xs_, ys_, 3, 3, ctx=tctx, batch_size=16, seed=7)
    out["small_train_snaps"] = np.stack(snaps)
    out["small_train_led"] = led(tctx.ledger.counts())

    # -- BASELINE configs ----------------------------------------------------
    A0, B0 = wl.config0()
    c0 = EmulatorContext(4096, 64, max_level=4)
    b0 = c0.ledger.snapshot()
    r = matmul.diag_abt(encoding.encode(c0, A0), encoding.encode(c0, B0, "vertical"))
    out["cfg0_out"] = encoding.decode(r)
    out["cfg0_led"] = led(c0.ledger.delta(b0))
    out["cfg0_level"] = np.array(r.level)

    X, W = wl.config1()
    c1 = EmulatorContext(32768, 128, max_level=12)
    b0 = c1.ledger.snapshot()
    r = matmul.diag_abt(encoding.encode(c1, X), encoding.encode(c1, W, "vertical"))
    out["cfg1_out"] = encoding.decode(r)
    out["cfg1_led"] = led(c1.ledger.delta(b0))
    out["cfg1_level"] = np.array(r.level)

    PY, X2 = wl.config2()
    for name, alev in (("rl", None), ("pru", 11)):
        c2 = EmulatorContext(32768, 128, max_level=12)
        r = matmul.diag_atb(encoding.encode(c2, PY, "horizontal", level=alev),
                            encoding.encode(c2, X2))
        out[f"cfg2_{name}_out"] = encoding.decode(r)
        out[f"cfg2_{name}_led"] = led(c2.ledger.counts())
        out[f"cfg2_{name}_level"] = np.array(r.level)

    Z3 = wl.config3()
    c3 = EmulatorContext(32768, 128, max_level=12, auto_bootstrap=True)
    r = approx.a_softmax(encoding.encode(c3, Z3, "horizontal"))
    out["cfg3_out"] = encoding.decode(r)
    out["cfg3_led"] = led(c3.ledger.counts())
    out["cfg3_level"] = np.array(r.level)

    X4, y4 = wl.config4()
    c4 = EmulatorContext(32768, 128, max_level=12, auto_bootstrap=True)
    snaps = training.run_steps(X4, y4, wl.CLASSES, 8, ctx=c4, batch_size=128,
                               lr=wl.LEARNING_RATE, seed=wl.INIT_SEED)
    out["cfg4_snaps"] = np.stack(snaps)
    out["cfg4_led"] = led(c4.ledger.counts())

    path = os.path.join(HERE, "hefit_golden.npz")
    # -- the two-party protocol end to end (training.py:159-338): fit with
    # validation logits and early stopping on unlearnable labels, so the
    # run exercises improved / continue / stop decisions (margins >= 4e-3)
    frng = np.random.default_rng(78)

    def draw(n):
        y = frng.integers(0, 3, n)
        x = frng.standard_normal((n, 12))
        return x / np.linalg.norm(x, axis=1, keepdims=True), y

    fxt, fyt = draw(48)
    fxv, fyv = draw(16)
    fctx = EmulatorContext(256, 16, max_level=12, auto_bootstrap=True)
    fr = training.fit(fxt, fyt, fxv, fyv, 3, ctx=fctx, lr=1.0, batch_size=16, epochs=8, patience=2, seed=1)
    out["fit_xt"], out["fit_yt"], out["fit_xv"], out["fit_yv"] = fxt, fyt, fxv, fyv
    out["fit_weights"] = fr.weights
    out["fit_val_losses"] = np.array(fr.val_losses)
    out["fit_train_losses"] = np.array(fr.train_losses)
    out["fit_meta"] = np.array([fr.epochs_run, fr.best_epoch, int(fr.stopped_early)])
    out["fit_led"] = led(fr.ledger_counts)

    np.savez_compressed(path, **out)
    print("wrote", path, "hefit", hefit.__version__, "numpy", np.__version__)


if __name__ == "__main__":
    main()
