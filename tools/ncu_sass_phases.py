"""Stall samples of one kernel split into phases at every BAR.SYNC (SASS order), from
`ncu -i REP --page source --csv --print-source=sass`.
usage: python tools/ncu_sass_phases.py sass.csv kernel-substring"""
import csv
import sys
from collections import Counter

csv.field_size_limit(1 << 30)
rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2]
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
    reasons = [(i, x) for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    tot = sum(float(r[i_s] or 0) for r in s["data"]) or 1
    print("==", s["name"][:100], "total samples", int(tot))
    ph, n = 0, 0
    acc, mix, ex, why = 0.0, Counter(), 0.0, Counter()
    def flush(tag):
        global acc, mix, ex, why
        top = ", ".join(f"{k.replace('stall_','')} {v/ max(acc,1)*100:.0f}%" for k, v in why.most_common(4))
        ops = ", ".join(f"{k} {int(v)}" for k, v in mix.most_common(6))
        print(f"  phase {ph:3d} ({tag:>8s}) instrs {n:5d}  samples {acc/tot*100:5.1f}%  warp-inst {ex/1e6:8.1f}M  [{top}]  {ops}")
        acc, mix, ex, why = 0.0, Counter(), 0.0, Counter()
    for r in s["data"]:
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        acc += float(r[i_s] or 0)
        ex += float(r[i_ex] or 0)
        for i, x in reasons:
            why[x] += float(r[i] or 0)
        mix[op] += 1
        n += 1
        if op.startswith("BAR") or op.startswith("EXIT"):
            flush(op[:8])
            ph += 1
            n = 0
    flush("end")
