"""Small end-to-end probe for compute-sanitizer: every fused kernel at N=2^16
(rotation, conjugation, mult + relin + rescale, plaintext/constant products,
level adjust, refresh) and a native schedule at N=2^9."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402

g = P.CKKSContext("cfg1", 128, seed=3)
z = np.random.default_rng(0).uniform(-1, 1, g.slot_count)
x = g.encrypt(z)
y = g.mult(g.lrot(x, 5), g.conj(x))
y = g.mult(y, z)
y = g.add(g.mult(y, 0.5), x)
y = g.bootstrap(g.level_adjust(y, 3))
err = float(np.max(np.abs(y.slots - (0.5 * np.roll(z, -5) * z * z + z))))
assert err < 1e-4, err
s = P.CKKSContext("small12", 16, seed=4, auto_bootstrap=True)
A = np.random.default_rng(1).uniform(-1, 1, (16, 16))
out = P.a_softmax(P.diag_abt(P.encode(s, A), P.encode(s, A[:4], "vertical")))
print("sanitize probe ok", err, out.level)
