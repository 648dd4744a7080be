#!/bin/bash
# r02ap: run-aligned chunk edges in backward pass 1 -- backward tests, timings on/off, trace
set -u
O=gpurun_out/${1:-r02ap}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_backward.py -m gpu -x -q > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 30 "$@" 2>>$O/err.log | tail -1 >> $O/al.jsonl; }
for rep in 1 2; do
for c in dlrm_small weak sweep_p8; do
  run --config $c
  run --config $c --opt bwd_aligned=0
done
done
run --config dlrm_wide --batches 4
run --config dlrm_wide --batches 4 --opt bwd_aligned=0
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 3 --warmup 3 > $O/ncu.log 2>&1
