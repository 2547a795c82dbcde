"""Diagnostic: config-4 epoch (8 x 128-row NAG steps) on the B200 context;
per step the max |imag| of W's slots and max |W - reference snapshot|."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import workloads as wl  # noqa: E402
from paper_2403_14111_b200.encoding import padded_array  # noqa: E402

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "hefit_golden.npz"))
X, y = wl.config4()
Y = P.one_hot(y, wl.CLASSES)
ctx = P.CKKSContext("cfg1", 128, seed=4, auto_bootstrap=True)
w0 = P.init_weights(wl.CLASSES, X.shape[1], wl.INIT_SEED)
W = P.encode(ctx, w0, "vertical")
st = P.TrainState(W, W)
for k in range(8):
    rows = slice(128 * k, 128 * k + 128)
    logits = P.nag_step(st, P.encode(ctx, X[rows]), P.encode(ctx, Y[rows], "horizontal"), wl.LEARNING_RATE, 128)
    lg = padded_array(logits)[:128, :10]
    probs = None
    full = padded_array(st.weights)[:10, :768]
    vfull = padded_array(st.momentum)[:10, :768]
    print(f"step {k + 1}: W level {st.weights.level} |imag W| {np.abs(full.imag).max():.2e} "
          f"|imag V| {np.abs(vfull.imag).max():.2e} |W-ref| {np.abs(full.real - g['cfg4_snaps'][k]).max():.2e} "
          f"|W| {np.abs(full.real).max():.2e} |imag logits| {np.abs(lg.imag).max():.2e}", flush=True)
