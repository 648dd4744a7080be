#!/bin/bash
# One GPU round trip: tests, smoke under ncu's launch list, bench line.  Outputs in gpurun_out/.
# usage: tools/gpu_check.sh TAG [pytest-args...]
set -u
TAG=${1:-run}; shift || true
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 "$@" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.log 2>&1
echo "smoke-under-ncu rc=$?" >> $O/smoke_ncu.log
timeout 900 python bench.py --out $O/bench.jsonl > $O/bench.log 2>&1
echo "bench rc=$?" >> $O/bench.log
