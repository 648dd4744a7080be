#!/bin/bash
# r02an: staged sub-batch rows in backward pass 1 -- backward tests, then timings on/off
set -u
O=gpurun_out/${1:-r02an}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_backward.py -m gpu -x -q > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 30 "$@" 2>>$O/err.log | tail -1 >> $O/stage.jsonl; }
for rep in 1 2; do
for c in dlrm_small sweep_p1; do
  run --config $c
  run --config $c --opt bwd_stage_rows=0
done
done
run --config weak --opt bwd_stage_rows=1
run --config weak
python tools/dbg/bwd_trace.py dlrm_small > $O/trace.txt 2>&1
