"""Outlier hunt: per-step device time of the bench pair over many steps
(synchronised per step, then free-running in groups of 10), plus the memory
pool's high-water marks (HC_POOL_STATS) when the context closes."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import _native as N  # noqa: E402
from paper_2403_14111_b200 import workloads as wl  # noqa: E402

os.environ.setdefault("HC_POOL_STATS", "1")
if os.environ.get("WITH_TORCH"):
    import torch
    torch.cuda.set_device(0)
    _keep = torch.empty(1, device="cuda")
smi = None
if os.environ.get("WITH_SMI"):
    import subprocess
    q = os.environ.get("SMI_QUERY", "clocks.sm,clocks.max.sm")
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader",
                            "-lms", "100"], stdout=subprocess.DEVNULL)
ctx = P.CKKSContext("cfg1", 128, seed=1)
X, W = wl.config1()
PY, _ = wl.config2()
EX, EW, EP = P.encode(ctx, X), P.encode(ctx, W, "vertical"), P.encode(ctx, PY, "horizontal")
L = N.lib()
ms = C.c_float()
for _ in range(3):
    P.diag_abt(EX, EW), P.diag_atb(EP, EX)
ctx.sync()
single = []
for i in range(30):
    N.check(L.hc_timer_begin(ctx._h))
    a = P.diag_abt(EX, EW)
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    t1 = ms.value
    N.check(L.hc_timer_begin(ctx._h))
    b = P.diag_atb(EP, EX)
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    single.append((round(t1, 1), round(ms.value, 1)))
groups = []
for i in range(6):
    N.check(L.hc_timer_begin(ctx._h))
    for _ in range(10):
        a, b = P.diag_abt(EX, EW), P.diag_atb(EP, EX)
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    groups.append(round(ms.value / 10, 2))
if smi:
    smi.terminate()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith(("HC_", "WITH_"))},
                  "single_abt_atb_ms": single, "free_running_10step_avg_ms": groups}), flush=True)
ctx.close()
