#!/bin/bash
# r02ay: chunk (bags per work unit) below the auto clamp of 32 at DLRM-small / weak
set -u
O=gpurun_out/${1:-r02ay}; mkdir -p $O
run() { timeout 300 python bench.py --no-cpu --no-alpha0 --no-backward --no-baseline --ag-leg 0 --steps 50 "$@" 2>>$O/err.log | tail -1 >> $O/chunk.jsonl; }
for rep in 1 2; do
for c in dlrm_small weak; do
  for ch in 0 16 20 24 28; do run --config $c --opt chunk=$ch; done
done
done
