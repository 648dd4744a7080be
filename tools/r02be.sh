#!/bin/bash
# r02be: bucket plan at DLRM-small with caps that hold its Zipf-hot bucket (~5 K keys)
set -u
O=gpurun_out/${1:-r02be}; mkdir -p $O
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 30 "$@" 2>>$O/err.log | tail -1 >> $O/bwd.jsonl; }
for rep in 1 2; do
  run --config dlrm_small --opt sort_mode=1
  for cap in 5632 6144 7168; do run --config dlrm_small --opt sort_mode=5 --opt bucket_cap=$cap; done
done
