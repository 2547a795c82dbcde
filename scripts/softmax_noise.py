"""Config-3 softmax: decrypted output vs the reference emulator's (noise-free)
output for several key / encryption seeds -- how much of the gap is CKKS noise."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import workloads as wl  # noqa: E402

gold = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "hefit_golden.npz"))["cfg3_out"]
Z = wl.config3()
for seed in (3, 4, 5, 6, 7, 8):
    ctx = P.CKKSContext("cfg1", 128, seed=seed, auto_bootstrap=True)
    out = P.decode(P.a_softmax(P.encode(ctx, Z, "horizontal")), tol=1e-2)
    d = np.abs(out - gold)
    print(f"seed {seed}: max |out - emulator| = {d.max():.3e}, rms = {np.sqrt((d ** 2).mean()):.3e}")
    del ctx
