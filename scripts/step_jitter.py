"""Per-step device time of the bench step, with/without nvidia-smi sampling running."""
import ctypes as C
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import _native as N  # noqa: E402
from paper_2403_14111_b200 import workloads as wl  # noqa: E402

ctx = P.CKKSContext("cfg1", 128, seed=1)
X, W = wl.config1()
PY, _ = wl.config2()
EX, EW, EP = P.encode(ctx, X), P.encode(ctx, W, "vertical"), P.encode(ctx, PY, "horizontal")
L = N.lib()
ms = C.c_float()
for mode in ("plain", "smi", "plain"):
    proc = None
    if mode == "smi":
        proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "100"],
                                stdout=subprocess.DEVNULL)
        time.sleep(0.5)
    out = []
    for i in range(8):
        N.check(L.hc_timer_begin(ctx._h))
        a = P.diag_abt(EX, EW)
        b = P.diag_atb(EP, EX)
        N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
        out.append(round(ms.value, 1))
    if proc:
        proc.terminate()
    print(mode, out)
