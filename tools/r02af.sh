#!/bin/bash
# r02af: ncu --set full of the cluster sort plan kernel (DLRM-small W=1)
set -u
O=gpurun_out/${1:-r02af}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bwd_cluster_sort -s 2 -c 1 \
  -o $O/cluster_full python bench.py --no-cpu --no-alpha0 --no-baseline --ag-leg 0 --steps 2 --warmup 3 --opt sort_mode=4 > $O/ncu.log 2>&1
echo "rc=$?" >> $O/ncu.log
