#!/bin/bash
# Round-2 GPU call: tests, smoke, bench lines (all configs + reference arm), ncu launch list of
# the default bench command (config 4), and ncu --set full captures of the config-4 layer
# kernels (one launch each).  Outputs go to gpurun_out/r02/ (summaries are copied into profiles/).
set -u
O=gpurun_out/r02
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?" >> $O/status
for c in 0 1 2 3; do
  timeout 900 python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err; echo "bench c$c rc=$?" >> $O/status
done
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench ref rc=$?" >> $O/status
# launch list of the default command (per-launch times are cold-cache and serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-side --no-ntt > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/status
# full captures: one launch of each config-4 layer kernel (after warm-up)
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"enc3_kernel|share3_kernel|planes_tc_kernel|mac_tc_kernel|mac_out_kernel|dec3_kernel" --launch-skip 25 -c 6 \
  -o /tmp/full_c4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-side --no-ntt > $O/ncu_full_c4.log 2>&1; echo "ncu full c4 rc=$?" >> $O/status
if [ -f /tmp/full_c4.ncu-rep ]; then
  ncu -i /tmp/full_c4.ncu-rep --page raw --csv > $O/full_c4_raw.csv 2>/dev/null
  ncu -i /tmp/full_c4.ncu-rep --page details --csv > $O/full_c4_details.csv 2>/dev/null
  python tools/ncu_traffic.py /tmp/full_c4.ncu-rep config4 $O/ncu_traffic.json > /dev/null 2>&1
  ncu -i /tmp/full_c4.ncu-rep --page source --csv --print-source sass > $O/full_c4_sass.csv 2>/dev/null
  rm -f /tmp/full_c4.ncu-rep
fi
cat $O/status
