#!/bin/bash
# r02ae: the cluster sort plan (sort_mode 4) -- parity tests, then backward timings vs the plain plan
set -u
O=gpurun_out/${1:-r02ae}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_backward.py -m gpu -x -q -k cluster > $O/pytest_cluster.log 2>&1
echo "rc=$?" >> $O/pytest_cluster.log
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 30 "$@" 2>>$O/err.log | tail -1 >> $O/bwd.jsonl; }
for c in dlrm_small weak sweep_p8 dlrm_wide; do
  run --config $c
  run --config $c --opt sort_mode=4
  run --config $c --opt sort_mode=4 --opt cluster_ctas=8
done
run --config dlrm_small --opt sort_mode=4 --opt cluster_ctas=4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
  python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 2 --warmup 3 --opt sort_mode=4 > $O/ncu.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_backward.py -m gpu -x -q > $O/pytest_bwd.log 2>&1
echo "rc=$?" >> $O/pytest_bwd.log
