"""Key-switch microbenchmark at BASELINE config 1 (N=2^16, top level).

Times R rotations of one level-12 ciphertext with CUDA events on the
library stream and prints key-switches/s plus the per-kernel breakdown of
one profiled rotation.  Small enough to run under ncu.

    python scripts/ks_micro.py [--reps 20] [--level 12] [--op rot|mult]
"""

import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2403_14111_b200 as P  # noqa: E402
from paper_2403_14111_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--level", type=int, default=12)
    ap.add_argument("--op", default="rot", choices=["rot", "mult"])
    ap.add_argument("--params", default="cfg1")
    a = ap.parse_args()
    ctx = P.CKKSContext(a.params, None, seed=3)
    L = N.lib()
    z = np.random.default_rng(0).uniform(-1, 1, ctx.slot_count)
    x = ctx.encrypt(z, a.level)

    def op():
        return ctx.lrot(x, 1) if a.op == "rot" else ctx.mult(x, x)

    for _ in range(3):
        op()
    ctx.sync()
    ms = C.c_float()
    N.check(L.hc_timer_begin(ctx._h))
    for _ in range(a.reps):
        op()
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    per = ms.value / a.reps
    N.check(L.hc_prof_begin(ctx._h))
    op()
    buf = C.create_string_buffer(1 << 16)
    N.check(L.hc_prof_end(ctx._h, buf, len(buf)))
    prof = json.loads(buf.value.decode())
    print(json.dumps({"op": a.op, "level": a.level, "ms_per_op": per, "ops_per_s": 1e3 / per,
                      "kernels": {k: [int(v[0]), round(v[1] * 1e3, 2), round(v[2] / max(v[1], 1e-9) / 1e6, 1)]
                                  for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
                      "legend": "kernel: [launches, total_us, algorithmic GB/s]"}))




def throughput(params="cfg1", level=12, reps=8):
    """Key switches per second with `s` concurrent independent chains."""
    ctx = P.CKKSContext(params, None, seed=3)
    x = ctx.encrypt(np.random.default_rng(0).uniform(-1, 1, ctx.slot_count), level)
    L = N.lib()
    out = {}
    for s in (1, 2, 4, 8, 16, 32):
        ms = C.c_float()
        N.check(L.hc_bench_keyswitch(ctx._h, x._h, s, reps, C.byref(ms)))
        out[s] = round(s * reps / (ms.value * 1e-3))
    return out


def batch_throughput(params="cfg1", level=12, reps=4):
    """Key switches per second: `s` concurrent chains, each rotating a batch of `b` operands per step."""
    ctx = P.CKKSContext(params, None, seed=3)
    x = ctx.encrypt(np.random.default_rng(0).uniform(-1, 1, ctx.slot_count), level)
    L = N.lib()
    out = {}
    for s in (1, 2, 4):
        for b in (1, 2, 4, 8, 16):
            ms = C.c_float()
            N.check(L.hc_bench_keyswitch_batch(ctx._h, x._h, s, b, reps, C.byref(ms)))
            out[f"s{s}_b{b}"] = round(s * b * reps / (ms.value * 1e-3))
    return out


def ntt_throughput(params="cfg1"):
    """Batched NTT: limb-transforms/s and GB/s (algorithmic 16N bytes per limb) vs limb count."""
    ctx = P.CKKSContext(params, None, seed=3)
    L = N.lib()
    out = {}
    for nl in (13, 51, 96, 512):
        for inv in (0, 1):
            ms = C.c_float()
            reps = 20
            N.check(L.hc_bench_ntt(ctx._h, nl, reps, inv, C.byref(ms)))
            per = ms.value / reps
            out[f"{'inv' if inv else 'fwd'}_{nl}"] = {"us": round(per * 1e3, 1),
                                                      "GBps": round(16 * ctx.N * nl / (per * 1e-3) / 1e9, 1)}
    return out


if __name__ == "__main__":
    if "--batch" in sys.argv:
        print(json.dumps({"keyswitch_per_s_streams_batch": batch_throughput(), "level": 12}))
    elif "--ntt" in sys.argv:
        print(json.dumps({"ntt": ntt_throughput()}))
    elif "--throughput" in sys.argv:
        lv = 12
        for a in sys.argv:
            if a.startswith("--level="):
                lv = int(a.split("=")[1])
        print(json.dumps({"keyswitch_per_s_by_streams": throughput(level=lv), "level": lv}))
    else:
        main()
