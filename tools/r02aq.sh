#!/bin/bash
# r02aq: L2 prefetch of a stage's rows by the consumers (option prefetch_rows)
set -u
O=gpurun_out/${1:-r02aq}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tunables or lane" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-backward --no-baseline --ag-leg 0 --steps 50 "$@" 2>>$O/err.log | tail -1 >> $O/pf.jsonl; }
for rep in 1 2; do
for c in dlrm_small weak sweep_p8 dlrm_wide; do
  run --config $c
  run --config $c --opt prefetch_rows=1
done
done
