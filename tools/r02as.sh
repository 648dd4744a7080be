#!/bin/bash
# r02as: the bucket sort plan (sort_mode 5) -- parity tests, then backward timings vs the plain plan
set -u
O=gpurun_out/${1:-r02as}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_backward.py -m gpu -x -q -k bucket > $O/pytest_bucket.log 2>&1
echo "rc=$?" >> $O/pytest_bucket.log
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 30 "$@" 2>>$O/err.log | tail -1 >> $O/bwd.jsonl; }
for rep in 1 2; do
for c in dlrm_small weak sweep_p1 sweep_p4; do
  run --config $c
  run --config $c --opt sort_mode=5
done
done
run --config sweep_p8 --opt sort_mode=5
run --config dlrm_wide --batches 4 --opt sort_mode=5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 3 --warmup 3 --opt sort_mode=5 > $O/ncu.log 2>&1
