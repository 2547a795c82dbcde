"""Instruction count per kernel in libhc_b200.so (static SASS), optionally by opcode."""
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else "."
out = subprocess.run(["cuobjdump", "-sass", "paper_2403_14111_b200/libhc_b200.so"], capture_output=True, text=True).stdout
cur, counts = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(.*", "", cur)
        counts[cur] = {}
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and cur:
        op = m.group(1).split(".")[0]
        counts[cur][op] = counts[cur].get(op, 0) + 1
for k, v in counts.items():
    if re.search(pat, k):
        tot = sum(n for o, n in v.items() if o not in ("NOP",))
        top = sorted(v.items(), key=lambda kv: -kv[1])[:8]
        print(f"{k:50s} total={tot:5d} " + " ".join(f"{o}={n}" for o, n in top))
