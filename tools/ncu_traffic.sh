#!/bin/bash
# DRAM traffic per launch of the fused kernel and of the backward kernel (pass 1) for every
# BASELINE config at W=1: one ncu capture each (serialised, cold caches: compare bytes, not time).
# Output: gpurun_out/ncu_<tag>/<config>{,_backward}.csv -> tools/ncu_traffic.py -> profiles/.
tag=${1:-r02}
O=gpurun_out/ncu_$tag
mkdir -p $O
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
for c in dlrm_small weak sweep_p1 sweep_p4 sweep_p8 sweep_p32 sweep_p128 dlrm_wide; do
  nb=4; [ $c = sweep_p128 ] && nb=2
  timeout 900 ncu --metrics $M --clock-control none -k regex:emb_a2a_kernel -s 3 -c 1 --csv \
    --log-file $O/$c.csv python bench.py --config $c --steps 3 --warmup 3 --batches $nb --no-cpu \
    --no-baseline --no-backward --no-alpha0 --ag-leg 0 > $O/$c.log 2>&1
  timeout 900 ncu --metrics $M --clock-control none -k regex:bwd_kernel -s 3 -c 1 --csv \
    --log-file $O/${c}_backward.csv python bench.py --config $c --steps 3 --warmup 3 --batches $nb \
    --no-cpu --no-baseline --no-alpha0 --ag-leg 0 > $O/${c}_backward.log 2>&1
  echo "done $c"
done
# f4: the fused AllGather + GEMM kernel (W = 1)
for c in ag_ffn ag_small; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:ag_gemm_kernel -s 3 -c 1 --csv \
    --log-file $O/$c.csv python bench.py --path ag_gemm --ag-config $c --steps 3 --warmup 2 \
    --no-cpu > $O/$c.log 2>&1
  echo "done $c"
done
