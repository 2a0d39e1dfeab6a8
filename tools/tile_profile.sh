#!/bin/bash
# ncu --set full capture of the three second-generation RNS tile kernels (one launch each,
# after warm-up) from tools/tile_ab.py's config-4 sub-batch; summaries into gpurun_out/tile/.
set -u
O=gpurun_out/tile
mkdir -p $O
timeout 300 python tools/tile_ab.py --images 256 --pack 2 --reps 3 > $O/ab.json 2> $O/ab.err; echo "ab rc=$?" > $O/status
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"enc3_kernel|share3_kernel|dec3_kernel" --launch-skip 9 -c 3 \
  -o /tmp/tile_full python tools/tile_ab.py --images 256 --pack 2 --reps 1 > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/status
if [ -f /tmp/tile_full.ncu-rep ]; then
  ncu -i /tmp/tile_full.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
  ncu -i /tmp/tile_full.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
  ncu -i /tmp/tile_full.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>/dev/null
  for k in enc3_kernel share3_kernel dec3_kernel; do python tools/ncu_sass_phases.py $O/sass.csv $k; done > $O/phases.txt 2>&1
  python tools/ncu_summary.py /tmp/tile_full.ncu-rep > $O/summary.md 2>&1
  rm -f /tmp/tile_full.ncu-rep
fi
cat $O/status
