"""Per-step device and host-issue time of the config-4 1024-row NAG step."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import _native as N  # noqa: E402
from paper_2403_14111_b200 import workloads as wl  # noqa: E402

L = N.lib()
X, y = wl.config4()
Y = P.one_hot(y, wl.CLASSES)
ctx = P.CKKSContext("cfg1", 128, seed=4, auto_bootstrap=True)
W = P.encode(ctx, P.init_weights(wl.CLASSES, X.shape[1], wl.INIT_SEED), "vertical")
EX, EY = P.encode(ctx, X), P.encode(ctx, Y, "horizontal")
state = P.TrainState(W, W)
ms = C.c_float()
rows = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    N.check(L.hc_timer_begin(ctx._h))
    t0 = time.perf_counter()
    P.nag_step(state, EX, EY, wl.LEARNING_RATE, X.shape[0])
    t1 = time.perf_counter()
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    rows.append((round(ms.value, 1), round((t1 - t0) * 1e3, 1)))
print("(device ms, host issue ms) per step:", rows)
