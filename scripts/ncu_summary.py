"""Print the headline sections of an ncu report (details page) and the top
warp-stall reasons (raw page) -- used to write the profiles/ summaries."""
import csv
import subprocess
import sys

KEYS = ['Throughput', 'Hit', 'Duration', 'Occupancy', 'Warp Cycles', 'Issue', 'Registers',
        'Shared Memory', 'Elapsed Cycles', 'SM Frequency']


def main(rep, kernel_filter=""):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    for r in csv.reader(det.splitlines()):
        if len(r) > 14 and kernel_filter in r[4] and any(k in r[12] for k in KEYS):
            print(f"{r[11][:28]:28s} | {r[12]} [{r[13]}] {r[14]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    for v in rows[2:]:
        if kernel_filter not in v[4]:
            continue
        st = []
        for k, x in zip(h, v):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(x.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1
        print("stalls:", ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in sorted(st, reverse=True)[:6]))
        for k, x in zip(h, v):
            if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                     "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
                     "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
                     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                     "smsp__inst_executed.sum"):
                print(f"{k} = {x}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
