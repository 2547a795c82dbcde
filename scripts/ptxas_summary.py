"""Registers / spills per kernel from the ptxas logs of the last build."""
import glob
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else "."
for log in sorted(glob.glob("paper_2403_14111_b200/csrc/build/*.ptxas.log")):
    name = None
    spill = ""
    for line in open(log):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
            name = re.sub(r"\(.*", "", name)
        m = re.search(r"(\d+) bytes spill stores", line)
        if m:
            spill = m.group(1)
        m = re.search(r"Used (\d+) registers", line)
        if m and name and re.search(pat, name):
            print(f"{name:60s} regs={m.group(1):4s} spill={spill}")
