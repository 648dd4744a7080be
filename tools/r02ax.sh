#!/bin/bash
# r02ax: bucket plan with a warp-aggregated bucket histogram
set -u
O=gpurun_out/${1:-r02ax}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_backward.py -m gpu -x -q -k bucket > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 30 "$@" 2>>$O/err.log | tail -1 >> $O/bwd.jsonl; }
for rep in 1 2; do
for c in dlrm_small weak sweep_p1 sweep_p4 sweep_p8; do
  run --config $c --opt sort_mode=5
  run --config $c --opt sort_mode=1
done
done
run --config dlrm_wide --batches 4 --opt sort_mode=5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 3 --warmup 3 --opt sort_mode=5 > $O/ncu.log 2>&1
