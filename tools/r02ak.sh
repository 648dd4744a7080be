#!/bin/bash
# r02ak: "l1_rows" -- forward parity, then auto vs forced on/off across configs
set -u
O=gpurun_out/${1:-r02ak}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-backward --no-baseline --ag-leg 0 --steps 50 "$@" 2>>$O/err.log | tail -1 >> $O/l1.jsonl; }
for c in dlrm_small weak sweep_p1 sweep_p4 sweep_p8 sweep_p32 dlrm_wide; do
  run --config $c
  run --config $c --opt l1_rows=0
  run --config $c --opt l1_rows=1
done
