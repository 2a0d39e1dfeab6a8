"""Group an ncu SASS source page by execution count (basic-block proxy): total warp
instructions per group and its opcode mix.  python tools/ncu_blocks.py X.csv [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ei = h.index("Source"), h.index("Instructions Executed")
byc = collections.defaultdict(list)
for r in rows[2:]:
    if len(r) > ei and r[ei].isdigit():
        byc[int(r[ei])].append(r[si].strip())
tot = sum(c * len(v) for c, v in byc.items())
for c, v in sorted(byc.items(), key=lambda kv: -kv[0] * len(kv[1]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 8]:
    ops = collections.Counter((x.split()[1] if x.split()[0].startswith("@") else x.split()[0]) for x in v)
    print(f"exec {c:>12,d} x {len(v):4d} = {100 * c * len(v) / tot:5.1f}%  {dict(ops.most_common(9))}")
