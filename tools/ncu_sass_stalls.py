"""Stall samples and instruction mix by SASS opcode per kernel, from
`ncu -i REP --page source --csv --print-source=sass`.  usage: python tools/ncu_sass_stalls.py sass.csv [kernel-substring]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "hdr": None, "data": []}
        secs.append(cur)
    elif cur is not None and cur["hdr"] is None:
        cur["hdr"] = r
    elif cur is not None and r:
        cur["data"].append(r)
for s in secs:
    if want not in s["name"]:
        continue
    h = s["hdr"]
    i_src, i_s, i_ex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    c, ex = Counter(), Counter()
    for r in s["data"]:
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        c[op] += float(r[i_s] or 0)
        ex[op] += float(r[i_ex] or 0)
    tot, tex = sum(c.values()) or 1, sum(ex.values()) or 1
    print("==", s["name"][:80])
    print("  stall samples by opcode:", [(k, round(v / tot * 100, 1)) for k, v in c.most_common(12)])
    print("  instruction mix:", [(k, round(v / tex * 100, 1)) for k, v in ex.most_common(14)])
    print("  warp instructions executed:", int(tex))
