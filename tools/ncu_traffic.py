"""Per-launch DRAM traffic of each kernel in an ncu --set full report, as the JSON that
bench.py's roofline.traffic reads:  python tools/ncu_traffic.py REP CONFIG OUT.json
(merges into OUT.json if it exists)."""
import csv
import io
import json
import os
import subprocess
import sys

rep, cfg, out = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = json.load(open(out)) if os.path.exists(out) else {}
d = res.setdefault(cfg, {})
for v in rows[2:]:
    name = v[h.index("Kernel Name")].split("<")[0].split("(")[0].replace("void ", "").split("::")[-1].strip()
    rd = float(v[h.index("dram__bytes_read.sum")]) * scale[units[h.index("dram__bytes_read.sum")]]
    wr = float(v[h.index("dram__bytes_write.sum")]) * scale[units[h.index("dram__bytes_write.sum")]]
    ms = float(v[h.index("gpu__time_duration.sum")]) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}[units[h.index("gpu__time_duration.sum")]]
    d[name] = {"dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr, "ncu_ms": ms,
               "kernel": v[h.index("Kernel Name")][:120]}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(d, indent=1))
