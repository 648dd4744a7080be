set -u
O=gpurun_out/r02l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ag_gemm_kernel -s 3 -c 1 -o $O/ag_pair_full python bench.py --path ag_gemm --steps 3 --warmup 2 --no-cpu > $O/ncu_full.log 2>&1; echo "ncu rc=$?" >> $O/ncu_full.log
