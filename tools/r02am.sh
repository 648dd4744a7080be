#!/bin/bash
# r02am: 16-bit L1 rows -- forward parity, then DLRM-wide bf16/f16 with L1 rows on/off
set -u
O=gpurun_out/${1:-r02am}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_variants.py -m gpu -x -q > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-backward --no-baseline --ag-leg 0 --steps 30 --batches 4 "$@" 2>>$O/err.log | tail -1 >> $O/h16.jsonl; }
for dt in bf16 f16; do
  run --config dlrm_wide --table-dtype $dt
  run --config dlrm_wide --table-dtype $dt --opt l1_rows=0
  run --config sweep_p32 --table-dtype $dt
  run --config sweep_p32 --table-dtype $dt --opt l1_rows=0
done
