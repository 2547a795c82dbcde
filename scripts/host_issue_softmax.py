"""Host-issue vs device time of the config-3 softmax (is the chain launch-bound?)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import _native as N  # noqa: E402
from paper_2403_14111_b200 import workloads as wl  # noqa: E402

ctx = P.CKKSContext("cfg1", 128, seed=3, auto_bootstrap=True)
EZ = P.encode(ctx, wl.config3(), "horizontal")
L = N.lib()
n0 = ctx.nonce
for _ in range(3):
    ctx.nonce = n0
    P.a_softmax(EZ)
ctx.sync()
for rep in range(4):
    ctx.nonce = n0
    l0 = L.hc_launch_count(ctx._h)
    t0 = time.perf_counter()
    out = P.a_softmax(EZ)
    t1 = time.perf_counter()
    ctx.sync()
    t2 = time.perf_counter()
    n = L.hc_launch_count(ctx._h) - l0
    print(f"host issue {1e3*(t1-t0):.2f} ms, wall {1e3*(t2-t0):.2f} ms, launches {n}, "
          f"{1e6*(t1-t0)/n:.2f} us/launch on the host")
