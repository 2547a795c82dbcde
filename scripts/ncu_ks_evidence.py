"""Turn an ncu --set full capture of one batched key-switch pipeline
(scripts/ks_batch_probe.py B 1 under --profile-from-start off) into the
evidence bench.py reports next to its roofline: DRAM bytes per key switch vs
the SURVEY §8(d) model (94.37 MB at level 12), and per-kernel issue activity.

    python scripts/ncu_ks_evidence.py RAW.csv[.gz] BATCH OUT.json [STEPS MODEL_BYTES BASIS]

With STEPS the capture is a ladder (scripts/ladder_probe.py): BATCH entries x
STEPS doubling steps, each charged MODEL_BYTES by the per-op model.
"""
import csv
import gzip
import io
import json
import sys

path, batch, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
model_arg = float(sys.argv[5]) if len(sys.argv) > 5 else None
basis_arg = sys.argv[6] if len(sys.argv) > 6 else None
raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
rows = list(csv.reader(io.StringIO(raw)))
h = {k: i for i, k in enumerate(rows[0])}
units = rows[1]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def nbytes(r, m):
    return float(r[h[m]]) * SCALE.get(units[h[m]], 1.0)
dram, us, inst = 0.0, 0.0, 0.0
issue = {}
for r in rows[2:]:
    name = r[h["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "").replace("hc::", "")
    if name == "ew_kernel":      # the probe's own bookkeeping, not the key switch
        continue
    b = nbytes(r, "dram__bytes_read.sum") + nbytes(r, "dram__bytes_write.sum")
    dram += b
    us += float(r[h["gpu__time_duration.sum"]])
    inst += float(r[h["smsp__inst_executed.sum"]])
    key = name + ("<" + r[h["Kernel Name"]].split("<")[1].split(">")[0] + ">" if "<" in r[h["Kernel Name"]] else "")
    issue.setdefault(key, []).append(round(float(r[h["sm__inst_issued.avg.pct_of_peak_sustained_active"]]), 1))
batch *= steps
per_ks = dram / batch
model = model_arg or 94.37e6
res = {"basis": basis_arg or f"ncu --set full of {batch} level-12 rotations (cfg1) in batched pipelines of 3 (scripts/ks_batch_probe.py), serialised, cold cache",
       "dram_bytes_per_keyswitch": per_ks, "model_bytes_per_keyswitch": model, "traffic_ratio": per_ks / model,
       "kernel_us_per_keyswitch": us / batch, "warp_instructions_per_keyswitch": inst / batch,
       "issue_active_pct": {k: v[0] if len(v) == 1 else v for k, v in issue.items()}}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
