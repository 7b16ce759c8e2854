"""Warp-stall breakdown and headline counters of one ncu report: python tools/ncu_stalls.py REP"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
d = dict(zip(rows[0], rows[2]))


def num(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


st = {k: num(k) for k in rows[0] if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")}
st = {k: v for k, v in st.items() if v}
tot = sum(st.values())
for k, x in sorted(st.items(), key=lambda a: -a[1])[:10]:
    print(f"{x / tot * 100:5.1f}% {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]:
    print(k, d.get(k))
