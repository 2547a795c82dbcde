"""Host-issue vs device time of one DiagABT/DiagATB pair (is the step launch-bound?)."""
import ctypes as C
import os
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
for _ in range(3):
    P.diag_abt(EX, EW); P.diag_atb(EP, EX)
ctx.sync()
for rep in range(3):
    n0 = L.hc_launch_count(ctx._h)
    t0 = time.perf_counter()
    a = P.diag_abt(EX, EW)
    b = P.diag_atb(EP, EX)
    t1 = time.perf_counter()
    ctx.sync()
    t2 = time.perf_counter()
    n = L.hc_launch_count(ctx._h) - n0
    print(f"host issue {1e3*(t1-t0):.2f} ms, wall {1e3*(t2-t0):.2f} ms, launches {n}, "
          f"{1e6*(t1-t0)/n:.2f} us/launch on the host")
