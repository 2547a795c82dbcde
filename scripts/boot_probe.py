"""CKKS bootstrapping at N = 2^16 (boot16): latency (CUDA events on the
library stream, after warm-up) and precision over several input ranges."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import _native as N  # noqa: E402

g = P.CKKSContext("boot16", 128, seed=5)
L = N.lib()
rng = np.random.default_rng(1)
out = {"params": "boot16: N=2^16, q0 60 + 12x42 (app) + 58,60,15x55 bits, P 4x60, top scale 2^55"}
errs = {}
for name, w in (("unit complex", rng.uniform(-1, 1, g.slot_count) + 1j * rng.uniform(-1, 1, g.slot_count)),
                ("real [-1,1]", rng.uniform(-1, 1, g.slot_count)),
                ("real [-128,128]", rng.uniform(-128, 128, g.slot_count)),
                ("real 1e-2", rng.uniform(-0.01, 0.01, g.slot_count))):
    x = g.encrypt(w, 0)
    y = g.ckks_bootstrap(x)
    d = y.slots - w
    errs[name] = {"max_abs": float(np.max(np.abs(d))), "mean_abs": float(np.mean(np.abs(d)))}
out["error"] = errs
x = g.encrypt(rng.uniform(-1, 1, g.slot_count), 0)
for _ in range(2):
    g.ckks_bootstrap(x)
g.sync()
ms = C.c_float()
reps = 5
N.check(L.hc_timer_begin(g._h))
for _ in range(reps):
    g.ckks_bootstrap(x)
N.check(L.hc_timer_end(g._h, C.byref(ms)))
out["ms_per_bootstrap"] = ms.value / reps
N.check(L.hc_prof_begin(g._h))
g.ckks_bootstrap(x)
buf = C.create_string_buffer(1 << 16)
N.check(L.hc_prof_end(g._h, buf, len(buf)))
prof = json.loads(buf.value.decode())
out["kernels_ms"] = {k: round(v[1], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:12]}
out["launches"] = int(sum(v[0] for v in prof.values()))
print(json.dumps(out, indent=1))
