"""One batched forward + inverse NTT over `nlimbs` limbs at N=2^16 (for ncu)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import _native as N  # noqa: E402

ctx = P.CKKSContext("cfg1", 128, seed=3)
ms = C.c_float()
for inv in (0, 1):
    N.check(N.lib().hc_bench_ntt(ctx._h, int(sys.argv[1]) if len(sys.argv) > 1 else 96, 1, inv, C.byref(ms)))
print("ok", ms.value)
