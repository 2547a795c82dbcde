"""Diagnostic: CKKS noise of single ops at config 1 (decrypted error in slots)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
g = P.CKKSContext(name, None, seed=5)
n = g.slot_count
rng = np.random.default_rng(1)
x = rng.uniform(-1, 1, n)
y = rng.uniform(-1, 1, n)


def err(ct, ref):
    v = ct.slots
    return f"re {np.abs(v.real - np.real(ref)).max():.2e} im {np.abs(v.imag - np.imag(ref)).max():.2e} lvl {ct.level}"


for lv in (g.max_level, g.max_level - 3):
    cx = g.encrypt(x, lv)
    cy = g.encrypt(y, lv)
    print("level", lv)
    print("  fresh      ", err(cx, x))
    print("  lrot 1     ", err(g.lrot(cx, 1), np.roll(x, -1)))
    print("  lrot 256   ", err(g.lrot(cx, 256), np.roll(x, -256)))
    print("  conj       ", err(g.conj(cx), x))
    print("  x+conj x   ", err(g.add(cx, g.conj(cx)), 2 * x))
    print("  mult       ", err(g.mult(cx, cy), x * y))
    print("  cmult .5   ", err(g.mult(cx, 0.5), 0.5 * x))
    a = cx
    ref = x.copy()
    for t in range(8):
        a = g.add(a, g.lrot(a, 1 << t))
        ref = ref + np.roll(ref, -(1 << t))
    print("  ladder 8   ", err(a, ref))
