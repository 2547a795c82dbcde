"""Summarise an ncu report: per kernel duration, DRAM bytes, throughput,
occupancy, pipe utilisation and the top stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}
want = [("dur_us", "gpu__time_duration.sum"), ("dram_rd_MB", "dram__bytes_read.sum"),
        ("dram_wr_MB", "dram__bytes_write.sum"), ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("issue_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        ("warps_act", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("regs", "launch__registers_per_thread"), ("grid", "launch__grid_size"),
        ("fma_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        ("alu_pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        ("fp64_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("l2_pct", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed")]
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0][:60]
    vals = []
    for short, m in want:
        v = r[col[m]] if m in col else "?"
        vals.append(f"{short}={v}")
    stalls = []
    for h, i in col.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    print(name, " ".join(vals), "stalls:", ", ".join(f"{n}={v:.2f}" for v, n in stalls[:4]))
