"""Ladders at cfg1 (for ncu and throughput): `streams` branches x batches of B
ciphertexts, `steps` doubling steps of stride 1 at level LEVEL, R repetitions.

usage: ladder_probe.py [B] [steps] [R] [streams] [level]
With HC_PROBE_PROFILE=1 only the measured run sits between
cudaProfilerStart / Stop (ncu --profile-from-start off)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import _native as N  # noqa: E402

arg = [int(v) for v in sys.argv[1:]]
B, steps, R, streams, level = (arg + [3, 2, 4, 1, 11][len(arg):])[:5]
ctx = P.CKKSContext("cfg1", None, seed=3)
x = ctx.encrypt(np.random.default_rng(0).uniform(-1, 1, ctx.slot_count) * 1e-3, level)
ms = C.c_float()
N.check(N.lib().hc_bench_ladder(ctx._h, x._h, streams, B, 1, steps, 1, C.byref(ms)))   # warm-up, key generation
prof = os.environ.get("HC_PROBE_PROFILE") == "1"
if prof:
    import torch
    torch.cuda.profiler.start()
N.check(N.lib().hc_bench_ladder(ctx._h, x._h, streams, B, 1, steps, R, C.byref(ms)))
if prof:
    torch.cuda.profiler.stop()
n = streams * B * R
print(f"ladders of {steps} steps: {n} in {ms.value:.3f} ms = {ms.value * 1e3 / n:.1f} us per ladder, "
      f"{ms.value * 1e3 / (n * steps):.1f} us per doubling step (B={B}, streams={streams}, level={level})")
