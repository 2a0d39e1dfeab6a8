"""gpurun_out/r02 (tools/round_profile_r02.sh) -> profiles/r02_*: bench lines, test log, ncu
launch list, full-capture CSVs, traffic JSON, and the markdown summary
(profiles/r02_ncu_summary.md).  python tools/collect_profiles.py"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
O, P = os.path.join(ROOT, "gpurun_out", "r02"), os.path.join(ROOT, "profiles")
for c in range(5):
    shutil.copy(f"{O}/bench_c{c}.json", f"{P}/r02_bench_config{c}.json")
for a, b in (("bench_ref.json", "r02_bench_reference_arm.json"), ("pytest_gpu.log", "r02_gpu_tests.log"),
             ("launches_c4.csv", "r02_launches_config4.csv"), ("full_c4_raw.csv", "r02_ncu_full_config4_raw.csv"),
             ("full_c4_details.csv", "r02_ncu_full_config4_details.csv"), ("ncu_traffic.json", "r02_ncu_traffic.json")):
    shutil.copy(f"{O}/{a}", f"{P}/{b}")
run = lambda *a: subprocess.run([sys.executable, *a], capture_output=True, text=True, cwd=ROOT).stdout
summ = run("tools/profile_summary.py", f"{O}/full_c4_raw.csv", f"{O}/full_c4_sass.csv",
           "config 4 (640 images per sub-batch: 128 ciphertext images of five 39x39 grids, 64->128, n=8192, 3-prime RNS): "
           "the six layer kernels")
ph = []
for k in ("enc3_kernel", "share3_kernel", "dec3_kernel"):
    seen = set()
    for line in run("tools/ncu_sass_phases.py", f"{O}/full_c4_sass.csv", k).splitlines():
        if line not in seen:
            seen.add(line)
            ph.append(line[:260])
b = json.load(open(f"{P}/r02_bench_config4.json"))
pk, step = b["roofline"]["per_kernel"], b["ms_per_step"]
share = lambda k: pk[k]["ms_per_launch"] * pk[k]["launches_per_step"] / step * 100
tr = json.load(open(f"{P}/r02_ncu_traffic.json"))["config4"]
rows = list(csv.reader(open(f"{O}/launches_c4.csv")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
kn, mv, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= mv:
        continue
    name = r[kn].split("<")[0].split("(")[0].replace("void ", "").split("::")[-1]
    tot[name] += float(r[mv].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r[mu], 1e-6)
    cnt[name] += 1
T = sum(tot.values())
ev = {"dec3_kernel": "dec_rns", "share3_kernel": "share", "mac_tc_kernel": "mac_tc", "enc3_kernel": "enc",
      "mac_out_kernel": "mac_out", "planes_tc_kernel": "planes_tc"}
lines, other, othern = [], 0.0, 0
for k, v in tot.most_common():
    if k in ev:
        lines.append(f"| {k} | {cnt[k]} | {v:.2f} | {v / T * 100:.1f}% | {share(ev[k]):.1f}% |")
    else:
        other += v
        othern += cnt[k]
lines.append(f"| probes (mma_i8_peak, imad_probe), weights3, torch fills, secret_kernel | {othern} | {other:.1f} | "
             f"{other / T * 100:.1f}% | outside the timed region |")
npass = open(f"{P}/r02_gpu_tests.log").read().strip().splitlines()[-1]
chunk = b["config"]["sub_batch_images"]
avg = b["config"]["images_per_gpu"] / round(pk["enc"]["launches_per_step"])
alg = lambda k: pk[k]["alg_bytes_per_launch"] / 1e9 * chunk / avg
fh = {}
raw = list(csv.reader(open(f"{O}/full_c4_raw.csv")))
i_f = raw[0].index("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed")
for r in raw[2:]:
    fh[r[raw[0].index("Kernel Name")].split("<")[0].replace("void ", "")] = float(r[i_f])
txt = f"""# Round 2 ncu summaries, final kernels (B200, sm_100a; tools/round_profile_r02.sh, one gpurun call)

Command profiled: `python bench.py` (default = config 4: 1024 images, 64->128, n = 8192, 3-prime RNS, five 39x39 grids per
ciphertext block; 2 sub-batches per step: 640 images = 128 ciphertext images, then 384 images = 77).  Bench lines of the same
call: `r02_bench_config*.json` (config 4: {b['value']:.0f} conv/s device, {b['e2e']['value']:.0f} e2e), reference arm
`r02_bench_reference_arm.json`, GPU tests `r02_gpu_tests.log` ({npass}).  The first capture of this round
(first-generation 1024-thread tile kernels, two 64x64 grids per block, 8245 conv/s) is kept as `r02a_*`; the SASS of the
butterfly passes with its opcode census is `r02_sass_butterfly.md`.  Regenerate with `python tools/collect_profiles.py`.

## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, r02_launches_config4.csv; cold-cache, serialised)

| kernel | launches | total ms | share | share in bench.py (CUDA events) |
|---|---|---|---|---|
""" + "\n".join(lines) + f"""

Only this repo's kernels run in the step; the shares agree with the live event timings of the bench line (under ncu the tile
kernels lose the overlap of HomShare with Enc on the second stream, hence their slightly larger share).

## Full captures (`ncu --set full --import-source on --clock-control none`, one launch per kernel after warm-up)

All six kernels of the 128-ciphertext sub-batch (640 images).

{summ}

DRAM traffic per launch (ncu) vs algorithmic bytes (bench.py accounting scaled to the 640-image sub-batch):
share3 {tr['share3_kernel']['dram_bytes'] / 1e9:.2f} / {alg('share'):.2f} GB, enc3 {tr['enc3_kernel']['dram_bytes'] / 1e9:.2f} / {alg('enc'):.2f},
dec3 {tr['dec3_kernel']['dram_bytes'] / 1e9:.2f} / {alg('dec_rns'):.2f}, planes_tc {tr['planes_tc_kernel']['dram_bytes'] / 1e9:.2f} / {alg('planes_tc'):.2f},
mac_tc {tr['mac_tc_kernel']['dram_bytes'] / 1e9:.2f} / {alg('mac_tc'):.2f}, mac_out {tr['mac_out_kernel']['dram_bytes'] / 1e9:.2f} / {alg('mac_out'):.2f} GB -- no kernel re-reads
(planes_tc reads 8-byte plane words in 32-byte sectors).

## Where the time goes inside the tile kernels (stall samples split at every BAR.SYNC, tools/ncu_sass_phases.py)

```
""" + "\n".join(ph) + f"""
```

Reading.  (1) All three tile kernels run two 512-thread CTAs per SM (warps active 49.5 %) and are bound by the FMA-heavy pipe:
{fh.get('dec3_kernel', 0):.1f} % (Dec), {fh.get('share3_kernel', 0):.1f} % (HomShare), {fh.get('enc3_kernel', 0):.1f} % (Enc) busy, math_pipe_throttle / not_selected the top stalls -- IMAD.WIDE
holds the pipe for two issue slots, so pipe busy exceeds issue active (55-58 %).  First generation (r02a): 46 %, 56 %, 64 %.
(2) Dec's phi pre-pass (phase 1) is about 10 % of its instructions and 16 % of its samples; in the first generation the same work,
fused into the first INTT pass, held 38 % of the samples.  (3) mac_tc is unchanged: FMA-heavy pipe {fh.get('mac_tc_kernel', 0):.1f} % busy in its
epilogue, tensor pipe about 40 %.
"""
open(f"{P}/r02_ncu_summary.md", "w").write(txt)
for c in range(5):
    d = json.load(open(f"{P}/r02_bench_config{c}.json"))
    print(c, round(d["value"], 1), d["unit"], round(d["ms_per_step"], 4), (d.get("e2e") or {}).get("value"),
          (d.get("cpu_baseline") or {}).get("value"))
print("per kernel", {k: (round(v["ms_per_launch"], 2), round(v.get("imad_frac", 0), 3), round(v.get("imad_frac_sass_floor", 0), 3),
                         round(v.get("hbm_frac", 0), 3), round(v.get("tensor_frac", 0), 3)) for k, v in pk.items()})
print("ref geometry", b["ref_geometry"]["value"], "pow2 packed", b["pow2_packed"]["value"], "config1", b["config1"]["value"],
      b["config1"]["grid39"]["value"], "ntt8192", b["ntt_n8192"]["fwd"]["transforms_per_s"], b["ntt_n8192"]["inv"]["transforms_per_s"])
print("reference arm", json.load(open(f"{P}/r02_bench_reference_arm.json"))["value"], fh)
