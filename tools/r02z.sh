set -u
O=gpurun_out/r02z2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python tools/ag_probe.py ag_ffn ab > $O/ab_ffn.log 2>&1
timeout 600 python tools/ag_probe.py ag_small ab > $O/ab_small.log 2>&1
for h in 0 1 4 5 7; do
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:ag_gemm_kernel -s 3 -c 1 --csv --log-file $O/traffic_h$h.csv python tools/ag_probe.py ag_ffn grid_h$h > $O/ncu_h$h.log 2>&1
done
