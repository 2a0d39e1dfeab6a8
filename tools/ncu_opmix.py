"""Executed-instruction mix and stall samples per opcode from an ncu source page:
ncu -i REP --page source --csv --print-source sass > X.csv; python tools/ncu_opmix.py X.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ei, wi = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ex, st = collections.Counter(), collections.Counter()
for r in rows[2:]:
    if len(r) <= ei:
        continue
    src = r[si].strip()
    if not src:
        continue
    toks = src.split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    if op.startswith("IMAD.WIDE"):
        op += " acc" if not src.rstrip(" ;").endswith("RZ") else " RZ"
    try:
        ex[op] += int(r[ei])
        st[op] += int(r[wi])
    except ValueError:
        pass
tot = sum(ex.values())
tots = sum(st.values())
print(f"total warp-instructions {tot:,}  stall samples {tots:,}")
for op, c in ex.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"  {op:24s} {c:16,d} {100 * c / tot:6.2f}%   samples {100 * st[op] / max(tots, 1):6.2f}%")
