#!/bin/bash
# r02bc: bucket plan with a batched bucket histogram, bucket_cap sweep (smem per CTA = 16 B x cap)
set -u
O=gpurun_out/${1:-r02bc}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_backward.py -m gpu -x -q -k bucket > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 30 "$@" 2>>$O/err.log | tail -1 >> $O/bwd.jsonl; }
for c in dlrm_small weak sweep_p1 sweep_p4; do
  run --config $c --opt sort_mode=1
  for cap in 1024 2048 4096 8192; do run --config $c --opt sort_mode=5 --opt bucket_cap=$cap; done
done
