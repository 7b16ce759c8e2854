"""Summarise ncu --set full captures (DRAM bytes, time, achieved GB/s, occupancy, IPC) into a
profiles/ table and update profiles/traffic.json (per-launch DRAM bytes read + written).
usage: python tools/ncu_summary.py OUT.txt CONFIG name=path.ncu-rep ..."""
import csv
import json
import os
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def main():
    out_txt, config = sys.argv[1], sys.argv[2]
    tpath = os.path.join(os.path.dirname(out_txt), "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    lines = ["# ncu --set full --clock-control none, one launch each (see profiles/README.md)",
             "# name | kernel | time us | DRAM read MB | DRAM write MB | DRAM GB/s | dram % of peak | regs | "
             "warps active % | IPC | warp instructions"]
    for arg in sys.argv[3:]:
        name, path = arg.split("=", 1)
        d, u = raw(path)

        def g(n):
            return float(d[n].replace(",", "")) * UNITS.get(u.get(n, ""), 1.0)

        rd, wr, t = g("dram__bytes_read.sum"), g("dram__bytes_write.sum"), g("gpu__time_duration.sum")
        traffic[f"{config}:{name}"] = rd + wr
        lines.append(f"{name:12s} {d['Kernel Name'][:46]:46s} {t * 1e6:8.1f} {rd / 1e6:8.1f} {wr / 1e6:8.1f} "
                     f"{(rd + wr) / t / 1e9:8.1f} {float(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):6.1f} "
                     f"{d['launch__registers_per_thread']:>4s} {float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):6.1f} "
                     f"{float(d['sm__inst_executed.avg.per_cycle_active']):5.2f} {d['smsp__inst_executed.sum']}")
    open(out_txt, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
