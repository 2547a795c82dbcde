"""Top SASS lines by warp-stall samples for one kernel of an ncu report, plus the
instruction mix weighted by execution count.

usage: ncu_sass_hot.py REPORT MANGLED_SUBSTRING [--full-op]
(the source page is dumped once for all kernels; the first section whose
mangled name contains the substring is analysed)"""
import csv
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
full_op = "--full-op" in sys.argv
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-kernel-base", "mangled"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
start = None
for i, r in enumerate(rows):
    if r and r[0] == "Kernel Name" and kern in r[1]:
        start = i
        break
if start is None:
    sys.exit(f"no kernel matching {kern}")
hdr = rows[start + 1]
ci = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[start + 2:]:
    if r and r[0] == "Kernel Name":
        break
    data.append(r)
mix = Counter()
tot_samples = 0
lines = []
for r in data:
    try:
        samp = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        ex = int(r[ci["Instructions Executed"]] or 0)
    except (ValueError, KeyError, IndexError):
        continue
    op = r[ci["Source"]].strip().split()
    op = [o for o in op if not o.startswith("@")]
    name = (op[0] if full_op else op[0].split(".")[0]) if op else "?"
    mix[name] += ex
    tot_samples += samp
    lines.append((samp, r[ci["Address"]], r[ci["Source"]].strip()[:70], ex))
tot_ex = sum(mix.values())
print("instruction mix (executed warp-instr):", tot_ex)
for k, v in mix.most_common(24 if full_op else 14):
    print(f"  {k:18s} {v:10d} {100*v/tot_ex:5.1f}%")
print("hottest lines by stall samples:")
for s, a, src, ex in sorted(lines, reverse=True)[:25]:
    print(f"  {100*s/max(tot_samples,1):5.1f}%  {src}")
