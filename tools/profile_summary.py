"""Markdown summary of exported ncu captures (raw page CSV + SASS source CSV):
python tools/profile_summary.py RAW.csv SASS.csv [title]"""
import collections
import csv
import sys

KEYS = [("gpu__time_duration.sum", "duration"),
        ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy pipe busy %"),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__registers_per_thread", "registers/thread"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
        ("smsp__inst_executed.sum", "warp instructions")]


def kshort(name):
    return name.replace("void ", "").split("(")[0].replace("ensei_gpu::", "")


raw = list(csv.reader(open(sys.argv[1])))
h, u = raw[0], raw[1]
title = sys.argv[3] if len(sys.argv) > 3 else sys.argv[1]
print(f"### {title}\n")
names = [kshort(r[h.index("Kernel Name")]) for r in raw[2:]]
print("| metric | " + " | ".join(names) + " |")
print("|---|" + "---|" * len(names))
for k, lab in KEYS:
    if k in h:
        i = h.index(k)
        print(f"| {lab} ({u[i]}) | " + " | ".join(r[i] for r in raw[2:]) + " |")
stalls = sorted({x for x in h if x.startswith("smsp__average_warps_issue_stalled") and x.endswith("per_issue_active.ratio")})
rows = []
for x in stalls:
    vals = []
    for r in raw[2:]:
        try:
            vals.append(float(r[h.index(x)]))
        except ValueError:
            vals.append(0.0)
    if max(vals) >= 0.3:
        rows.append((max(vals), x, vals))
for _, x, vals in sorted(rows, reverse=True)[:8]:
    lab = x.replace("smsp__average_warps_issue_stalled_", "stall ").replace("_per_issue_active.ratio", "")
    print(f"| {lab} (per issue) | " + " | ".join(f"{v:.2f}" for v in vals) + " |")
print()
if len(sys.argv) > 2:
    rows = list(csv.reader(open(sys.argv[2])))
    # one SASS table per kernel: header rows start with "Kernel Name" in the source export
    blocks, cur, hdr, kn = [], None, None, None
    for r in rows:
        if r and r[0] == "Kernel Name":
            kn = kshort(r[1]) if len(r) > 1 else "?"
            continue
        if r and "Source" in r and "Instructions Executed" in r:
            hdr = r
            cur = collections.Counter()
            blocks.append((kn, cur))
            continue
        if hdr and cur is not None and len(r) > hdr.index("Instructions Executed"):
            src = r[hdr.index("Source")].strip()
            n = r[hdr.index("Instructions Executed")]
            if src and n.isdigit():
                t = src.split()
                op = t[1] if t[0].startswith("@") else t[0]
                cur[op] += int(n)
    seen = set()
    for kn, c in blocks:
        tot = sum(c.values())
        if not tot or kn in seen:
            continue
        seen.add(kn)
        top = ", ".join(f"{op} {100 * v / tot:.1f}%" for op, v in c.most_common(8))
        print(f"- `{kn}` executed-instruction mix: {top}")
    print()
