#!/bin/bash
# r02aj: L1 policy of the forward's row loads (no_allocate / allocate / evict_last), interleaved
set -u
O=gpurun_out/${1:-r02aj}; mkdir -p $O
run() { local lib=$1; shift; timeout 300 python bench.py --no-cpu --no-alpha0 --no-backward --no-baseline --ag-leg 0 --steps 50 "$@" 2>>$O/err.log | tail -1 | sed "s|^|$lib |" >> $O/l1.txt; }
for rep in 1 2; do
for c in dlrm_small weak sweep_p8 dlrm_wide; do
  for lib in paper_2305_06942_b200/libemba2a.so variants/l1alloc/libemba2a.so variants/l1last/libemba2a.so; do
    run $lib --config $c
  done
done
done
