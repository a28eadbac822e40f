"""Summarise ncu reports (raw page) into the numbers DESIGN.md / bench.py cite.
Usage: python scripts/ncu_summary.py REPORT.ncu-rep [...]  (run where ncu is installed)"""
import csv
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_shared_mem", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active"]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    for v in rows[2:]:
        d = {k: (u, x) for k, u, x in zip(head, units, v)}
        print(f"== {path}: {d.get('Kernel Name', ('', '?'))[1][:100]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k][1]:>16s} {d[k][0]}")
        st = []
        for k, (u, x) in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    st.append((float(x.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1
        print("  stall samples: " + ", ".join(f"{k} {x / tot * 100:.0f}%" for x, k in sorted(st, reverse=True)[:7]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summarise(p)
