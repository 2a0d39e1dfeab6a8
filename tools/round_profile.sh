#!/bin/bash
# One GPU call: tests, smoke, bench lines (all configs + reference arm), ncu launch list of
# the default bench command, and ncu --set full captures of the config-1 kernels and the
# config-4 MAC.  Outputs go to gpurun_out/round/ (summaries are copied into profiles/).
set -u
O=gpurun_out/round
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status
timeout 900 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err; echo "bench c1 rc=$?" >> $O/status
for c in 0 2 3 4; do
  timeout 900 python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err; echo "bench c$c rc=$?" >> $O/status
done
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench ref rc=$?" >> $O/status
# launch list of the same default command (per-launch times are cold-cache and serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/status
# full captures: one launch of each config-1 layer kernel (after warm-up) and the config-4 MAC
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"tile_enc_kernel|share_kernel|mac_kara_kernel|dec_kernel" --launch-skip 8 -c 4 \
  -o /tmp/full_c1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_full_c1.log 2>&1; echo "ncu full c1 rc=$?" >> $O/status
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"mac_i8p|mac_kara" --launch-skip 2 -c 1 \
  -o /tmp/full_c4_mac python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_full_c4.log 2>&1; echo "ncu full c4 rc=$?" >> $O/status
# export the captures as CSV (raw metrics + SASS source with per-instruction counters), drop the .ncu-rep
for r in full_c1 full_c4_mac; do
  if [ -f /tmp/$r.ncu-rep ]; then
    ncu -i /tmp/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
    ncu -i /tmp/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>/dev/null
    python tools/ncu_traffic.py /tmp/$r.ncu-rep $( [ $r = full_c1 ] && echo config1 || echo config4 ) $O/ncu_traffic.json > /dev/null 2>&1
    ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass > $O/${r}_sass.csv 2>/dev/null
    rm -f /tmp/$r.ncu-rep
  fi
done
cat $O/status
