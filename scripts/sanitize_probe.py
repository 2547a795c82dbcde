"""Small end-to-end probe for compute-sanitizer: every fused kernel at N=2^16
(rotation, conjugation, hoisted rotations, mult + relin + rescale, product
sum, plaintext/constant products, level adjust, refresh), asynchronous
transfers, and native schedules at N=2^9 (multi-block lockstep softmax with
batched refreshes)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import _native as N  # noqa: E402

g = P.CKKSContext("cfg1", 128, seed=3)
z = np.random.default_rng(0).uniform(-1, 1, g.slot_count)
x = g.encrypt(z)
y = g.mult(g.lrot(x, 5), g.conj(x))
y = g.mult(y, z)
y = g.add(g.mult(y, 0.5), x)
y = g.bootstrap(g.level_adjust(y, 3))
err = float(np.max(np.abs(y.slots - (0.5 * np.roll(z, -5) * z * z + z))))
assert err < 1e-4, err
h = g.lrot_hoisted(x, [1, 7, 0, 300])
s3 = g.mult_sum([x, h[0], h[1]], [h[1], x, h[3]])
want = z * np.roll(z, -7) + np.roll(z, -1) * z + np.roll(z, -7) * np.roll(z, -300)
assert float(np.max(np.abs(s3.slots - want))) < 1e-3
res = np.ascontiguousarray(x.residues())
hh = C.c_void_p()
N.check(N.lib().hc_ct_upload_async(g._h, res.ctypes.data_as(N.U64P), x.level, C.byref(hh)))
up = P.Ciphertext(g, hh)
sq = g.mult(up, up)
out = np.zeros((2, sq.level + 1, g.N), np.uint64)
N.check(N.lib().hc_ct_download_async(sq._h, out.ctypes.data_as(N.U64P)))
g.sync()
assert np.array_equal(out, g.mult(x, x).residues())
s = P.CKKSContext("small12", 16, seed=4, auto_bootstrap=True)
A = np.random.default_rng(1).uniform(-1, 1, (48, 16))
sm = P.a_softmax(P.diag_abt(P.encode(s, A), P.encode(s, A[:4], "vertical")))
print("sanitize probe ok", err, sm.level)
