"""Benchmark of the HETAL hot path on B200 (BASELINE.json metric).

One step = DiagABT (config 1: X 128x768 times W^T, W 10x768 vertically tiled,
period 16) followed by DiagATB (config 2: (P-Y)^T X, RL branch), RNS-CKKS at
N = 2^16, 58 + 12x42 | 3x60 bits, dnum 4, Delta 2^42, on one 128-row block
pair.  With N GPUs the pair's c/2 = 8 independent diagonal passes are
sharded round-robin over the ranks; each rank's partial accumulators are
mod-summed over NCCL (all-reduce + hc_mod_reduce on the library stream)
before the replicated conj epilogue -- strong scaling, bit-exact to 1 GPU.
Inputs are encrypted (client side) before timing and stay resident in HBM;
the switching keys alone (2.3 GB) exceed L2, so no flush is needed between
steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload pair|train|softmax|table4]

value = ms per DiagABT+DiagATB pair for the whole job (lower is better).
roofline = the step's algorithmic HBM bytes under SURVEY §8(d)'s per-op
model (accumulated by the library op by op) over the step time, against the
measured HBM peak.  e2e = the same through the public API with host buffers:
the step's input ciphertexts are copied host->device from pinned memory and
its outputs device->host inside the timed region.  --impl reference times
whole pairs on the C RNS-CKKS oracle (the reference itself has no CKKS; its
float64 slot emulator is timed beside it) on the host cores.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DiagABT/DiagATB ms at N=2^16 (128x768, 16 cls); key-switch/s; % HBM roofline"
CONFIG = {"workload": "DiagABT cfg1 (128x768 . (16x768)^T) + DiagATB-RL cfg2 ((128x16)^T . 128x768)",
          "ring": "N=2^16", "moduli": "58+12x42 | 3x60 bits", "dnum": 4, "scale": "2^42",
          "grid": "128x256", "classes": 10, "period": 16, "block_rows_per_rank": 128,
          "l2": "no flush: switching keys (2.3 GB) > 126 MB L2 are streamed every step"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.lines = device, None, []

    def start(self):
        if os.environ.get("HC_BENCH_NO_SMI"):    # diagnosis only: no clock evidence
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_ready(self, timeout=5.0):
        """nvidia-smi's start-up (NVML init) can stall the process's CUDA calls
        for a few hundred ms: start the sampler before warm-up and let its
        first sample arrive before the timed region."""
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.05)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def quiet_gc():
    """A full cyclic-GC pass over the process (torch alone brings ~10^5
    objects) stalls the issuing thread for 100+ ms and starves the GPU of
    work: freeze the objects that exist after set-up and collect the rest
    only between measurements (the library's ciphertext handles are not
    cyclic, so reference counting frees them)."""
    import gc
    gc.collect()
    gc.freeze()
    if os.environ.get("HC_BENCH_GC", "0") != "1":
        gc.disable()


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world == 1 and os.environ.get("HC_BENCH_TORCH_EARLY", "1") == "1":
        # bring torch's CUDA state up before the library context exists, not
        # lazily at the first barrier next to the timed region
        import torch
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            torch.cuda.synchronize()
    if world > 1:
        import torch
        import torch.distributed as dist
        ndev = torch.cuda.device_count()
        local = local % max(ndev, 1)
        torch.cuda.set_device(local)
        # HC_DIST_BACKEND=gloo lets the multi-rank plumbing run with several ranks
        # on one device (functional check only; timings are then meaningless)
        backend = os.environ.get("HC_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def _coll_device():
    import torch.distributed as dist
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def all_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def all_sum(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], device=_coll_device(), dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def keyswitch_rate(ctx, ct, streams=4, batch=16, reps=4):
    """Key switches per second of batched level-12 rotations (hc_bench_keyswitch_batch)."""
    from paper_2403_14111_b200 import _native as N
    ms = C.c_float()
    N.check(N.lib().hc_bench_keyswitch_batch(ctx._h, ct._h, streams, batch, 1, C.byref(ms)))   # warm
    N.check(N.lib().hc_bench_keyswitch_batch(ctx._h, ct._h, streams, batch, reps, C.byref(ms)))
    return streams * batch * reps / (ms.value * 1e-3)


def ladder_rate(ctx, ct, streams=3, batch=3, steps=8, reps=2):
    """Doubling steps per second of the column ladder (stride 1, `steps`
    steps: radix-4 rotate-and-sum stages with the fused forms on) over
    `streams` concurrent batches of `batch` level-11 ciphertexts
    (hc_bench_ladder) -- the op the DiagABT / DiagATB passes are made of."""
    from paper_2403_14111_b200 import _native as N
    ms = C.c_float()
    N.check(N.lib().hc_bench_ladder(ctx._h, ct._h, streams, batch, 1, steps, 1, C.byref(ms)))   # warm
    N.check(N.lib().hc_bench_ladder(ctx._h, ct._h, streams, batch, 1, steps, reps, C.byref(ms)))
    return streams * batch * steps * reps / (ms.value * 1e-3)


def ncu_evidence(name="ncu_keyswitch.json"):
    """DRAM traffic and issue utilisation of the key-switch pipeline (or, with
    ncu_ladder.json, of the radix-4 ladder stage) from the committed
    ncu --set full captures under profiles/r2/."""
    path = os.path.join(ROOT, "profiles", "r2", name)
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU legs: the C RNS-CKKS oracle (the same CKKS computation, all host
# threads) and the reference's own float64 slot emulator (hefit, 1 core, no
# cryptography).  Timed on whole DiagABT + DiagATB-RL pairs.
# ---------------------------------------------------------------------------


def oracle_pairs(budget_s, max_pairs):
    """Whole pairs (DiagABT cfg1 + DiagATB-RL cfg2, every pass, prologue and
    conj epilogue) on the C RNS-CKKS oracle with OpenMP over all host
    threads.  The switching keys are generated before timing (the GPU arm's
    keys are resident too); pairs are timed until `budget_s` or `max_pairs`.
    Returns (per-pair ms list, setup s)."""
    # torchrun exports OMP_NUM_THREADS=1; the CPU leg uses every host thread
    # (read by libgomp when the oracle library loads)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())
    from oracle import rns as R
    from oracle import slots as S
    from paper_2403_14111_b200 import workloads as wl
    from paper_2403_14111_b200.matmul import rotation_steps

    t0 = time.perf_counter()
    X, W = wl.config1()
    PY, _ = wl.config2()
    o = R.OracleCKKSContext("cfg1", 128, seed=1)
    OX, OW, OP = S.encode(o, X), S.encode(o, W, "vertical"), S.encode(o, PY, "horizontal")
    steps = set(rotation_steps(o, "diag_abt", 16)) | set(rotation_steps(o, "diag_atb", 16))
    for r in sorted(steps):
        o.p.key(o.p.galois(r))
    o.p.key(0)
    o.p.key(2 * o.p.N - 1)
    setup = time.perf_counter() - t0
    ms = []
    t_start = time.perf_counter()
    while len(ms) < max_pairs and (not ms or time.perf_counter() - t_start + ms[-1] / 1e3 < budget_s):
        t1 = time.perf_counter()
        S.diag_abt(OX, OW)
        S.diag_atb(OP, OX)
        ms.append((time.perf_counter() - t1) * 1e3)
    return ms, setup


def emulator_pair(reps=3):
    """The reference's own CPU path: hefit's float64 slot emulator (no
    cryptography; numpy element-wise complex ops, single-threaded) running
    the same pair at the same shapes.  None when hefit is not installed
    (baseline/_ref)."""
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(k, "1")
    p = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(p, "hefit")) and p not in sys.path:
        sys.path.append(p)
    try:
        import hefit
    except Exception:
        return None
    from paper_2403_14111_b200 import workloads as wl
    X, W = wl.config1()
    PY, _ = wl.config2()
    ms = []
    for _ in range(reps + 1):
        e = hefit.EmulatorContext(32768, 128, max_level=12)
        EX, EW = hefit.encode(e, X), hefit.encode(e, W, "vertical")
        EP = hefit.encode(e, PY, "horizontal")
        t0 = time.perf_counter()
        hefit.diag_abt(EX, EW)
        hefit.diag_atb(EP, EX)
        ms.append((time.perf_counter() - t0) * 1e3)
    return {"value": statistics.median(ms[1:]), "unit": "ms", "cores": 1, "kind": "reference",
            "sample": f"hefit {getattr(hefit, '__version__', '?')} float64 slot emulator (the reference's own CPU "
                      f"path, no cryptography), whole pair, median of {reps} after 1 warm-up"}


def run_reference(args, world, rank):
    if rank != 0:
        return
    cores = os.cpu_count()
    # a few minutes at most: whole pairs until ~90 s of timed CPU work
    ms, setup = oracle_pairs(budget_s=float(os.environ.get("HC_REF_BUDGET_S", "90")), max_pairs=max(1, args.steps))
    v = statistics.median(ms)
    emu = emulator_pair()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "ms", "n_gpus": args.gpus,
            "steps": len(ms), "warmup": 0, "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": v, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": CONFIG,
            "timed_s": round(sum(ms) / 1e3, 1), "setup_s": round(setup, 1), "runs_ms": [round(x, 1) for x in ms],
            "cpu_baseline": {"value": v, "unit": "ms", "cores": cores, "kind": "port",
                             "sample": f"{len(ms)} whole DiagABT cfg1 + DiagATB-RL cfg2 pairs (all 8 passes, "
                                       "prologue and conj epilogue) on the C RNS-CKKS oracle, OpenMP over all "
                                       "host threads; switching keys generated before timing; median"},
            "reference_emulator": emu,
            "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def run_b200(args, world, rank, local):
    import torch

    import paper_2403_14111_b200 as P
    from paper_2403_14111_b200 import _native as N
    from paper_2403_14111_b200 import workloads as wl

    L = N.lib()
    # every rank holds the same keys and inputs; with N > 1 the pair's c/2 = 8
    # diagonal passes are sharded round-robin over the ranks and the partial
    # accumulators are mod-summed over NCCL (SURVEY §8(e) k-diagonal sharding)
    ctx = P.CKKSContext("cfg1", 128, seed=1, device=local)
    if world > 1:
        from paper_2403_14111_b200 import sharding
        ctx.set_pass_shard(world, rank, sharding.NcclModReducer())
    X, W = wl.config1()
    PY, _ = wl.config2()
    EX, EW, EP = P.encode(ctx, X), P.encode(ctx, W, "vertical"), P.encode(ctx, PY, "horizontal")

    def step():
        logits = P.diag_abt(EX, EW)
        grad = P.diag_atb(EP, EX)
        return logits, grad

    clocks = Clocks(local)
    clocks.start()
    clocks.wait_ready()
    for _ in range(args.warmup):
        step()
    ctx.sync()
    quiet_gc()
    counts0 = ctx.ledger.counts()
    extra0 = ctx.extra
    model0 = ctx.model_bytes()
    launches0 = L.hc_launch_count(ctx._h)
    barrier(world)
    N.check(L.hc_timer_begin(ctx._h))
    outs = None
    trace = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        outs = step()
        trace.append(round((time.perf_counter() - t0) * 1e3, 1))
    ms = C.c_float()
    t0 = time.perf_counter()
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    trace.append(("drain", round((time.perf_counter() - t0) * 1e3, 1)))
    barrier(world)
    clk = clocks.stop()
    total_ms = all_max(ms.value, world)
    launches = L.hc_launch_count(ctx._h) - launches0
    counts = {k: v - counts0[k] for k, v in ctx.ledger.counts().items()}
    ks = ctx.extra["KeySwitch"] - extra0["KeySwitch"]
    model_step = all_sum(ctx.model_bytes() - model0, world) / args.steps
    ks = int(all_sum(ks, world))
    ms_step = total_ms / args.steps
    value = ms_step                    # whole job: one pair per step (passes sharded over the ranks)

    # one profiled step, serialised on one stream so each kernel's CUDA-event
    # duration is its own (concurrent branches would overlap the intervals)
    ctx.set_streams(1)
    N.check(L.hc_prof_begin(ctx._h))
    step()
    buf = C.create_string_buffer(1 << 16)
    N.check(L.hc_prof_end(ctx._h, buf, len(buf)))
    prof = json.loads(buf.value.decode())
    ctx.set_streams(8)
    # time per product in a separate pass
    N.check(L.hc_timer_begin(ctx._h))
    P.diag_abt(EX, EW)
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    abt_ms = ms.value
    N.check(L.hc_timer_begin(ctx._h))
    P.diag_atb(EP, EX)
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    atb_ms = ms.value

    # e2e through the public API with pinned host buffers
    inputs = [b for b in EX.flat() + EW.flat() + EP.flat()]
    host_in = []
    for b in inputs:
        r = b.residues()
        t = torch.empty(r.size, dtype=torch.int64, pin_memory=True)
        t.numpy()[:] = r.ravel().view(np.int64)
        host_in.append((t, b.level))
    lg, gr = outs
    out_shapes = [(2, b.level + 1, ctx.N) for b in lg.flat() + gr.flat()]
    host_out = [torch.empty(int(np.prod(s)), dtype=torch.int64, pin_memory=True) for s in out_shapes]
    h2d = sum(t.numel() * 8 for t, _ in host_in)
    d2h = sum(t.numel() * 8 for t in host_out)
    e2e_steps = max(1, args.steps)

    def upload(t, lv):
        h = C.c_void_p()
        N.check(L.hc_ct_upload_async(ctx._h, C.cast(C.c_void_p(t.data_ptr()), N.U64P), lv, C.byref(h)))
        return P.Ciphertext(ctx, h)

    def e2e_step():
        # asynchronous transfers on the library's copy streams: the upload of
        # the DiagATB operand overlaps DiagABT, each product's download
        # overlaps the next work, and step i+1's uploads overlap step i
        cts = [upload(t, lv) for t, lv in host_in[:6]]
        gX = P.EncodedMatrix(ctx, (tuple(cts[0:3]),), EX.shape, "none", None)
        gW = P.EncodedMatrix(ctx, (tuple(cts[3:6]),), EW.shape, "vertical", EW.period)
        a = P.diag_abt(gX, gW)
        gP = P.EncodedMatrix(ctx, ((upload(*host_in[6]),),), EP.shape, "horizontal", EP.period)
        for blk, t in zip(a.flat(), host_out):
            N.check(L.hc_ct_download_async(blk._h, C.cast(C.c_void_p(t.data_ptr()), N.U64P)))
        g = P.diag_atb(gP, gX)
        for blk, t in zip(g.flat(), host_out[len(a.flat()):]):
            N.check(L.hc_ct_download_async(blk._h, C.cast(C.c_void_p(t.data_ptr()), N.U64P)))

    # untimed warm-up (the copy-stream allocations reach their working set),
    # then three timed runs of `steps` end-to-end steps; the median is reported
    for _ in range(args.warmup):
        e2e_step()
    ctx.sync()
    e2e_runs = []
    for _ in range(3):
        barrier(world)
        N.check(L.hc_timer_begin(ctx._h))
        for _ in range(e2e_steps):
            e2e_step()
        N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
        barrier(world)
        e2e_runs.append(all_max(ms.value, world) / e2e_steps)
    e2e_ms = statistics.median(e2e_runs)
    # the end-to-end results are the resident run's, bit for bit
    e2e_exact = all(np.array_equal(t.numpy().view(np.uint64), blk.residues().ravel())
                    for blk, t in zip(lg.flat() + gr.flat(), host_out))

    hbm, peak_kind = peaks()
    # level-12 key-switch throughput (batched rotations of one top-level
    # ciphertext; the §8(d) per-op model charges 94.37 MB per switch)
    ks_rate = keyswitch_rate(ctx, EX.flat()[0])
    ks_model = 94.37e6
    # a doubling-ladder step add(x, lrot(x, 2^t)) at level 11 (the level of
    # DiagABT's first ladder): Rot 4 Lq + 2 d (Lq + K) plus Add 6 Lq limbs
    x11 = ctx.encrypt(np.zeros(ctx.slot_count), 11)
    lad_rate = ladder_rate(ctx, x11)
    lad_model = (4 * 12 + 2 * 3 * (12 + 3) + 6 * 12) * 8.0 * ctx.N
    # the dominant kernel of the profiled step (its own algorithmic bytes per
    # launch over its CUDA-event time), for the breakdown
    top = max(prof.items(), key=lambda kv: kv[1][1])
    name, (n_launch, k_ms, k_bytes) = top
    step_prof_ms = sum(v[1] for v in prof.values())
    ncu = ncu_evidence()
    ncu_lad = ncu_evidence("ncu_ladder.json")
    achieved = model_step / (ms_step * 1e-3) / 1e9
    peak_all = hbm * world
    line = {
        "metric": METRIC, "value": value, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded, BASELINE configs 1-2)",
        "config": dict(CONFIG, parallelism=f"diagonal passes sharded over {world} rank(s), NCCL mod-sum"
                       if world > 1 else "1 GPU"),
        "diag_abt_ms": abt_ms, "diag_atb_ms": atb_ms,
        # key-switch/s = the ledger's (Rot + Conj + Mult) per second;
        # the pipelines actually run (one ModUp + ModDown each) are fewer: a
        # radix-4 rotate-and-sum stage stands for two ladder rotations and a
        # product sum for its n relinearisations
        "keyswitch_per_s": (counts["Rot"] + counts["Conj"] + counts["Mult"]) / (total_ms * 1e-3),
        "ledger_per_step": {k: v // args.steps for k, v in counts.items()},
        "keyswitch_ops_per_step": (counts["Rot"] + counts["Conj"] + counts["Mult"]) // args.steps,
        "keyswitch_pipelines_per_step": ks // args.steps,
        # algorithmic bytes of the step under the per-op model
        # (inputs read once, outputs written once, key-switch intermediates on
        # chip), accumulated by the library op by op at each op's level
        "roofline": {"bound": "hbm", "basis": "SURVEY 8(d) per-op model of the whole step",
                     "achieved": achieved, "peak": peak_all, "unit": "GB/s", "frac": achieved / peak_all,
                     "peak_kind": peak_kind, "model_bytes_per_step": model_step,
                     "traffic": ncu.get("dram_bytes_per_keyswitch") if ncu else None,
                     "traffic_ratio": ncu.get("traffic_ratio") if ncu else None,
                     "traffic_basis": ncu.get("basis") if ncu else None},
        "keyswitch_level12": {"per_s": ks_rate, "model_bytes": ks_model,
                              "achieved_gbs": ks_rate * ks_model / 1e9,
                              "frac": ks_rate * ks_model / 1e9 / hbm,
                              "sample": "4 streams x batches of 16 rotations of one level-12 ciphertext"},
        "ladder_level11": {"doubling_steps_per_s": lad_rate, "model_bytes": lad_model,
                           "achieved_gbs": lad_rate * lad_model / 1e9, "frac": lad_rate * lad_model / 1e9 / hbm,
                           "sample": "3 streams x batches of 3 level-11 ciphertexts, 8-step column ladders "
                                     "(4 radix-4 rotate-and-sum stages each)",
                           "traffic": ncu_lad.get("dram_bytes_per_keyswitch") if ncu_lad else None,
                           "traffic_ratio": ncu_lad.get("traffic_ratio") if ncu_lad else None,
                           "traffic_basis": ncu_lad.get("basis") if ncu_lad else None},
        "issue_active_pct": ncu.get("issue_active_pct") if ncu else None,
        "dominant_kernel": {"name": name, "launches_per_step": int(n_launch), "ms_per_step": k_ms,
                            "achieved_gbs": k_bytes / (k_ms * 1e-3) / 1e9,
                            "share_of_step": k_ms / step_prof_ms},
        "kernel_breakdown_ms": {k: round(v[1], 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
            # per kernel: [launches, ms, algorithmic GB/s] of the serialised profiled step
            "kernel_detail": {k: [int(v[0]), round(v[1], 3), round(v[2] / max(v[1], 1e-9) / 1e6, 1)]
                              for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
        "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "transfers": "async copy streams (hc_ct_upload_async / hc_ct_download_async)",
                "runs_ms": [round(v, 3) for v in e2e_runs], "statistic": "median of 3 timed runs after warm-up",
                "residues_equal_resident_run": bool(e2e_exact)},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if os.environ.get("HC_BENCH_TRACE"):
        line["host_issue_ms_per_step"] = trace
    if world == 1 and not args.no_cpu:
        ms_cpu, _ = oracle_pairs(budget_s=1.0, max_pairs=1)
        line["cpu_baseline"] = {"value": ms_cpu[0], "unit": "ms", "cores": os.cpu_count(), "kind": "port",
                                "sample": "one whole DiagABT cfg1 + DiagATB-RL cfg2 pair (all 8 passes, prologue, "
                                          "conj epilogue) on the C RNS-CKKS oracle, OpenMP over all host threads, "
                                          "keys generated before timing",
                                "reference_emulator": emulator_pair()}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_train_step(args, world, rank, local):
    """BASELINE config 4 as a data-parallel NAG step: the 1024-row batch's 8
    block rows are sharded over ranks; the DiagATB block-row pre-sums are
    mod-summed across ranks (NCCL) -- strong scaling (fixed 1024 rows/step)."""
    import paper_2403_14111_b200 as P
    from paper_2403_14111_b200 import _native as N
    from paper_2403_14111_b200 import sharding
    from paper_2403_14111_b200 import workloads as wl

    L = N.lib()
    X, y = wl.config4()
    Y = P.one_hot(y, wl.CLASSES)
    ctx = P.CKKSContext("boot16" if args.boot == "ckks" else "cfg1", 128, seed=4, device=local, auto_bootstrap=True,
                        bootstrap=args.boot)
    w0 = P.init_weights(wl.CLASSES, X.shape[1], wl.INIT_SEED)
    W = P.encode(ctx, w0, "vertical")                       # replicated, same nonces on all ranks
    ctx.nonce = sharding.rank_nonce_base(rank) + 1000
    Xl = sharding.local_rows(X, 128, world, rank)
    Yl = sharding.local_rows(Y, 128, world, rank)
    EX, EY = P.encode(ctx, Xl), P.encode(ctx, Yl, "horizontal")
    red = sharding.NcclModReducer() if world > 1 else None
    state = P.TrainState(W, W)

    def step():
        P.nag_step(state, EX, EY, wl.LEARNING_RATE, X.shape[0], reducer=red)

    clocks = Clocks(local)
    clocks.start()
    clocks.wait_ready()
    for _ in range(args.warmup):
        step()
    ctx.sync()
    quiet_gc()
    c0 = ctx.ledger.counts()
    launches0 = L.hc_launch_count(ctx._h)
    barrier(world)
    ms = C.c_float()
    N.check(L.hc_timer_begin(ctx._h))
    for _ in range(args.steps):
        step()
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    barrier(world)
    clk = clocks.stop()
    total = all_max(ms.value, world)
    counts = {k: (v - c0[k]) // args.steps for k, v in ctx.ledger.counts().items()}
    # one profiled step (kernel time per kernel, streams serialised)
    ctx.set_streams(1)
    N.check(L.hc_prof_begin(ctx._h))
    step()
    buf = C.create_string_buffer(1 << 16)
    N.check(L.hc_prof_end(ctx._h, buf, len(buf)))
    prof = json.loads(buf.value.decode())
    ctx.set_streams(8)
    hbm, _ = peaks()
    line = {"metric": "NAG training step ms, config 4 (1024 rows x 768, 10 classes, N=2^16)",
            "value": total / args.steps, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total / args.steps, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded 10-class Gaussian mixture, BASELINE config 4)",
            "config": {"workload": "data-parallel NAG step over 8 block rows of 128 (DiagABT, softmax, "
                                   "DiagATB with cross-rank mod-sum, NAG update, refresh)",
                       "refresh": "CKKS bootstrapping (boot16 chain)" if args.boot == "ckks"
                       else "surrogate (decrypt/re-encrypt), not CKKS bootstrapping",
                       "rows": int(X.shape[0]), "block_rows_per_rank": len(sharding.partition(8, world, rank))},
            "ledger_per_step": counts, "gpu_launches": int(L.hc_launch_count(ctx._h) - launches0),
            "kernel_breakdown_ms": {k: round(v[1], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
            # per kernel: [launches, ms, algorithmic GB/s] of the serialised profiled step
            "kernel_detail": {k: [int(v[0]), round(v[1], 3), round(v[2] / max(v[1], 1e-9) / 1e6, 1)]
                              for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
            "clocks": clk}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_softmax(args, world, rank, local):
    """BASELINE config 3: the encrypted softmax approximation of one 128x16
    logit block (10 active classes) at N=2^16, the reference's SoftmaxConfig
    defaults (approx.py:51-57) and per-operand auto-bootstrap (refresh
    surrogate).  One dependent ciphertext chain: replicas only for N > 1."""
    import paper_2403_14111_b200 as P
    from paper_2403_14111_b200 import _native as N
    from paper_2403_14111_b200 import workloads as wl

    L = N.lib()
    Z = wl.config3()
    ctx = P.CKKSContext("boot16" if args.boot == "ckks" else "cfg1", 128, seed=3, device=local, auto_bootstrap=True,
                        bootstrap=args.boot)
    EZ = P.encode(ctx, Z, "horizontal")
    nonce0 = ctx.nonce

    def step():
        ctx.nonce = nonce0   # same refresh nonces every step
        return P.a_softmax(EZ)

    clocks = Clocks(local)
    clocks.start()
    clocks.wait_ready()
    for _ in range(args.warmup):
        out = step()
    ctx.sync()
    ez = np.exp(Z - Z.max(axis=1, keepdims=True))
    err = float(np.max(np.abs(P.decode(out, tol=1e-2) - ez / ez.sum(axis=1, keepdims=True))))
    quiet_gc()
    c0 = ctx.ledger.counts()
    launches0 = L.hc_launch_count(ctx._h)
    barrier(world)
    ms = C.c_float()
    N.check(L.hc_timer_begin(ctx._h))
    for _ in range(args.steps):
        out = step()
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    barrier(world)
    clk = clocks.stop()
    total = all_max(ms.value, world)
    counts = {k: (v - c0[k]) // args.steps for k, v in ctx.ledger.counts().items()}
    N.check(L.hc_prof_begin(ctx._h))
    step()
    buf = C.create_string_buffer(1 << 16)
    N.check(L.hc_prof_end(ctx._h, buf, len(buf)))
    prof = json.loads(buf.value.decode())
    line = {"metric": "encrypted softmax ms, config 3 (128x16 logits, 10 classes, N=2^16)",
            "value": total / args.steps, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total / args.steps, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded U[-128,128] logits, BASELINE config 3)",
            "config": {"workload": "a_softmax (domain extension R=8 L=2 n=5, a_max, a_exp, a_inv) on one block; "
                                   "replicas only for N > 1",
                       "refresh": "CKKS bootstrapping (boot16 chain)" if args.boot == "ckks"
                       else "surrogate (decrypt/re-encrypt), not CKKS bootstrapping"},
            "max_abs_err_vs_float64": err, "ledger_per_step": counts,
            "kernel_breakdown_ms": {k: round(v[1], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
            # per kernel: [launches, ms, algorithmic GB/s] of the serialised profiled step
            "kernel_detail": {k: [int(v[0]), round(v[1], 3), round(v[2] / max(v[1], 1e-9) / 1e6, 1)]
                              for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
            "gpu_launches": int(L.hc_launch_count(ctx._h) - launches0), "clocks": clk}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_bootstrap(args, world, rank, local):
    """One CKKS bootstrapping of a level-0 ciphertext at
    N = 2^16 on the boot16 chain (ModRaise, CoeffToSlot, EvalMod,
    SlotToCoeff) landing at level 12; replicas only for N > 1.  The paper's
    HEaaN bootstrapping: 159 ms on an A40."""
    import paper_2403_14111_b200 as P
    from paper_2403_14111_b200 import _native as N

    L = N.lib()
    ctx = P.CKKSContext("boot16", 128, seed=5, device=local)
    rng = np.random.default_rng(1)
    w = rng.uniform(-1, 1, ctx.slot_count) + 1j * rng.uniform(-1, 1, ctx.slot_count)
    x = ctx.encrypt(w, 0)
    clocks = Clocks(local)
    clocks.start()
    clocks.wait_ready()
    for _ in range(args.warmup):
        y = ctx.ckks_bootstrap(x)
    ctx.sync()
    err = float(np.max(np.abs(y.slots - w)))
    quiet_gc()
    launches0 = L.hc_launch_count(ctx._h)
    barrier(world)
    ms = C.c_float()
    N.check(L.hc_timer_begin(ctx._h))
    for _ in range(args.steps):
        y = ctx.ckks_bootstrap(x)
    N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
    barrier(world)
    clk = clocks.stop()
    total = all_max(ms.value, world)
    N.check(L.hc_prof_begin(ctx._h))
    ctx.ckks_bootstrap(x)
    buf = C.create_string_buffer(1 << 16)
    N.check(L.hc_prof_end(ctx._h, buf, len(buf)))
    prof = json.loads(buf.value.decode())
    line = {"metric": "CKKS bootstrapping ms (N=2^16, 2^15 slots, level 0 -> 12)",
            "value": total / args.steps, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total / args.steps, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic (uniform complex slots)",
            "config": {"workload": "ModRaise + CoeffToSlot (3 BSGS levels) + EvalMod (Chebyshev 27, 4 double "
                                   "angles, x2) + SlotToCoeff (3 levels); replicas only for N > 1",
                       "chain": "q0 60 + 12x42 (app) + 58, 60, 15x55 bits; P 4x60; dnum 8"},
            "max_abs_err": err, "paper_hea_an_a40_ms": 159.0,
            "kernel_breakdown_ms": {k: round(v[1], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
            # per kernel: [launches, ms, algorithmic GB/s] of the serialised profiled step
            "kernel_detail": {k: [int(v[0]), round(v[1], 3), round(v[2] / max(v[1], 1e-9) / 1e6, 1)]
                              for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
            "gpu_launches": int(L.hc_launch_count(ctx._h) - launches0), "clocks": clk}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_table4(args, world, rank, local):
    """The paper's Table 4 (reference harness cli.py:240-356):
    DiagABT vs the column-major baseline and DiagATB vs the row-major
    baseline on encrypted operands at N = 2^16 with the table's shapes
    (a, b, c) and the reference harness's grid (2^15 slots, s0 = min(next
    pow2(a), slots) rows).  Device time per call (median of `steps` // 4 + 1
    calls after one warm-up); replicas only.  The paper's A40 / HEaaN times
    (seconds) are carried for comparison."""
    import paper_2403_14111_b200 as P
    from paper_2403_14111_b200 import _native as N

    L = N.lib()
    rng = np.random.default_rng(7)
    # (a, b, c) and the paper's A40 seconds: ColMajor, DiagABT, RowMajor, DiagATB
    table = [((128, 128, 4), (0.1104, 0.0601, 0.1171, 0.0415)),
             ((256, 256, 8), (0.3203, 0.1211, 0.3167, 0.1239)),
             ((512, 769, 4), (0.7609, 0.1223, 0.7176, 0.3343)),
             ((1024, 769, 8), (3.0428, 0.3710, 2.8546, 1.2558)),
             ((2048, 769, 16), (12.6251, 1.2376, 11.8220, 4.9970))]
    if os.environ.get("HC_TABLE4_QUICK"):
        table = table[:2]
    rows = []
    ms = C.c_float()

    def timed(fn, reps):
        fn()
        N.check(L.hc_timer_begin(ctx._h))
        for _ in range(reps):
            fn()
        N.check(L.hc_timer_end(ctx._h, C.byref(ms)))
        return ms.value / reps

    clocks = Clocks(local)
    clocks.start()
    clocks.wait_ready()
    for (a, b, c), paper in table:
        s0 = min(1 << (a - 1).bit_length(), 32768)
        ctx = P.CKKSContext("cfg1", s0, seed=11, device=local)
        A = rng.uniform(-1, 1, (a, b)) / np.sqrt(b)
        B = rng.uniform(-1, 1, (c, b)) / np.sqrt(b)
        Y = rng.uniform(-1, 1, (a, c))
        EA, EBv, EB = P.encode(ctx, A), P.encode(ctx, B, "vertical"), P.encode(ctx, B)
        EY, EYu = P.encode(ctx, Y, "horizontal"), P.encode(ctx, Y)
        reps = max(1, args.steps // 4) if a <= 512 else 1
        t_abt = timed(lambda: P.diag_abt(EA, EBv), reps)
        t_cm = timed(lambda: P.col_major_abt(EA, EB), reps)
        t_atb = timed(lambda: P.diag_atb(EY, EA), reps)
        t_rm = timed(lambda: P.row_major_atb(EYu, EA), reps)
        rows.append({"shape": [a, b, c], "grid_rows": s0, "diag_abt_ms": t_abt, "col_major_abt_ms": t_cm,
                     "abt_speedup": t_cm / t_abt, "diag_atb_ms": t_atb, "row_major_atb_ms": t_rm,
                     "atb_speedup": t_rm / t_atb,
                     "paper_a40_s": {"col_major": paper[0], "diag_abt": paper[1], "row_major": paper[2],
                                     "diag_atb": paper[3]},
                     "vs_paper_a40": {"diag_abt": paper[1] * 1e3 / t_abt, "diag_atb": paper[3] * 1e3 / t_atb}})
        del EA, EBv, EB, EY, EYu
        ctx.close()
    clk = clocks.stop()
    line = {"metric": "Table 4: DiagABT / DiagATB vs column- / row-major baselines, ms per encrypted matmul "
                      "(N=2^16)", "value": rows[-1]["diag_abt_ms"] + rows[-1]["diag_atb_ms"], "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": 1, "ms_per_step": rows[-1]["diag_abt_ms"] + rows[-1][
                "diag_atb_ms"], "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (uniform, rows scaled 1/sqrt(b))",
            "config": {"workload": "Table 4 shapes (a, b, c); cfg1 parameters, grid rows min(next_pow2(a), 2^15)",
                       "shapes": [t[0] for t in table]},
            "rows": rows, "clocks": clk}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="pair", choices=["pair", "train", "softmax", "bootstrap", "table4"],
                    help="pair: DiagABT+DiagATB (BASELINE metric); train: config-4 data-parallel NAG step; "
                         "softmax: config-3 encrypted softmax; bootstrap: one CKKS bootstrapping at N=2^16; "
                         "table4: the paper's Table-4 matmul comparison")
    ap.add_argument("--boot", default="surrogate", choices=["surrogate", "ckks"],
                    help="train / softmax: the reference's bootstrap as the refresh surrogate or real CKKS "
                         "bootstrapping (boot16 chain)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, world, rank)
        return
    world, rank, local = dist_setup(args.gpus)
    if args.workload == "train":
        run_train_step(args, world, rank, local)
    elif args.workload == "softmax":
        run_softmax(args, world, rank, local)
    elif args.workload == "bootstrap":
        run_bootstrap(args, world, rank, local)
    elif args.workload == "table4":
        run_table4(args, world, rank, local)
    else:
        run_b200(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
