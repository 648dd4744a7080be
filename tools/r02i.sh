set -u
O=gpurun_out/r02i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_smoke.py > $O/san_$t.log 2>&1; echo "rc=$?" >> $O/san_$t.log
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_smoke.py --W 2 > $O/san_memcheck_W2.log 2>&1; echo "rc=$?" >> $O/san_memcheck_W2.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.log 2>&1; echo "rc=$?" >> $O/smoke_ncu.log
