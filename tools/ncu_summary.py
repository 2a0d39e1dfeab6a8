"""Key metrics of every kernel in an .ncu-rep (ncu -i REP --page raw --csv)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
for v in rows[2:]:
    print("==", v[h.index("Kernel Name")][:90])
    for k in KEYS:
        if k in h:
            print(f"   {k:70s} {v[h.index(k)]:>16s} {u[h.index(k)]}")
    st = [(float(v[i]), h[i]) for i in range(len(h))
          if h[i].startswith("smsp__average_warps_issue_stalled") and h[i].endswith("per_issue_active.ratio")
          and v[i] not in ("", "n/a")]
    for val, name in sorted(st, reverse=True)[:7]:
        print(f"   stall {name.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {val:.2f}")
