"""One stream of batched rotations at cfg1 level 12 (for ncu): batch B, reps R.

With HC_PROBE_PROFILE=1 a warm-up pipeline runs first and only the measured
one sits between cudaProfilerStart / Stop (ncu --profile-from-start off)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import _native as N  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 3
R = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ctx = P.CKKSContext("cfg1", None, seed=3)
x = ctx.encrypt(np.random.default_rng(0).uniform(-1, 1, ctx.slot_count), 12)
ms = C.c_float()
N.check(N.lib().hc_bench_keyswitch_batch(ctx._h, x._h, 1, B, 1, C.byref(ms)))   # warm-up, key generation
prof = os.environ.get("HC_PROBE_PROFILE") == "1"
if prof:
    import torch
    torch.cuda.profiler.start()
N.check(N.lib().hc_bench_keyswitch_batch(ctx._h, x._h, 1, B, R, C.byref(ms)))
if prof:
    torch.cuda.profiler.stop()
print("key switches/s", round(B * R / (ms.value * 1e-3)))
