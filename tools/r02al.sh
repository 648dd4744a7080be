#!/bin/bash
# r02al: SM-affine chunk order x L1 rows at DLRM-small / weak / sweep_p8
set -u
O=gpurun_out/${1:-r02al}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tunables or lane" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-backward --no-baseline --ag-leg 0 --steps 50 "$@" 2>>$O/err.log | tail -1 >> $O/aff.jsonl; }
for rep in 1 2; do
for c in dlrm_small weak sweep_p8; do
  run --config $c
  run --config $c --opt sm_affine=1
  run --config $c --opt sm_affine=1 --opt l1_rows=1
  run --config $c --opt sm_affine=1 --opt l1_rows=0
done
done
