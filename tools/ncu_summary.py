"""One-screen summary of an ncu --set full report (first profiled kernel):
duration, DRAM bytes, throughput, occupancy, issue and stall figures."""
import csv
import subprocess
import sys


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return {h: (v, u) for h, u, v in zip(r[0], r[1], r[2])}


KEYS = [
    ("Kernel Name", "Kernel Name"),
    ("duration", "gpu__time_duration.sum"),
    ("dram read", "dram__bytes_read.sum"),
    ("dram write", "dram__bytes_write.sum"),
    ("dram % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 hit %", "lts__t_sector_hit_rate.pct"),
    ("L1 hit %", "l1tex__t_sector_hit_rate.pct"),
    ("registers/thread", "launch__registers_per_thread"),
    ("theoretical occupancy %", "sm__maximum_warps_per_active_cycle_pct"),
    ("achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue slots busy %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("fp64 pipe %", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
]

if __name__ == "__main__":
    d = raw(sys.argv[1])
    for label, key in KEYS:
        if key in d:
            v, u = d[key]
            print(f"{label:26s} {v} {u}")
    stalls = sorted(((float(v.replace(",", "")), k) for k, (v, u) in d.items()
                     if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                     and v not in ("", "n/a")), reverse=True)[:6]
    print("top stalls (warps per issue):", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}"
                                                     for v, k in stalls))
