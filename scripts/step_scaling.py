"""Average step time of the bench pair vs the number of back-to-back steps
(one device timer around K steps, host running ahead), with and without the
nvidia-smi clock sampler and Python's garbage collector."""
import ctypes as C
import gc
import os
import subprocess
import sys
import time

if os.environ.get("WITH_TORCH"):
    import torch
    torch.cuda.init()
    _keep = torch.empty(1, device="cuda")
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


def run(k):
    N.check(L.hc_timer_begin(ctx._h))
    t0 = time.perf_counter()
    for _ in range(k):
        a = P.diag_abt(EX, EW)
        b = P.diag_atb(EP, EX)
    t1 = time.perf_counter()
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    return round(ms.value / k, 2), round((t1 - t0) * 1e3 / k, 2)


for _ in range(3):
    run(1)
for mode in ("plain", "smi", "nogc", "plain"):
    proc = None
    if mode == "smi":
        proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "100"],
                                stdout=subprocess.DEVNULL)
        time.sleep(0.5)
    if mode == "nogc":
        gc.disable()
    res = {k: run(k) for k in (1, 2, 5, 10, 20)}
    gc.enable()
    if proc:
        proc.terminate()
    print(mode, "{K: (device ms/step, host issue ms/step)}", res, flush=True)
