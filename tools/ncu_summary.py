"""Summarise an ncu report (raw page): time, DRAM bytes, pipe utilisation, top stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
units = dict(zip(hdr, rows[1]))
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    print("kernel:", d.get("Kernel Name", "")[:90])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg"]:
        print("  ", k, d.get(k), units.get(k, ""))
    st = []
    for h, v in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                st.append((float(v.replace(",", "")), h))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    for x, h in sorted(st, reverse=True)[:8]:
        print("   %5.1f%% %s" % (100 * x / tot, h.replace("smsp__pcsamp_warps_issue_stalled_", "stall_")))
