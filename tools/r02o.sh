set -u
O=gpurun_out/r02o; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for m in 1 3; do
  timeout 600 python tools/bwd_probe.py dlrm_small weak --opt sort_mode=$m > $O/probe_m$m.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_m$m.csv -k regex:bwd_ python tools/bwd_probe.py dlrm_small weak --reps 2 --batches 2 --opt sort_mode=$m > $O/ncu_m$m.log 2>&1
done
