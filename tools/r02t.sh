set -u
O=gpurun_out/r02t; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:emb_a2a_kernel -s 12 -c 1 -o $O/fwd_p1 python bench.py --config sweep_p1 --batches 8 --steps 6 --warmup 3 --no-cpu --no-baseline --no-backward --no-alpha0 --ag-leg 0 > $O/ncu_p1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:emb_a2a_kernel -s 12 -c 1 -o $O/fwd_small python bench.py --config dlrm_small --steps 6 --warmup 3 --no-cpu --no-baseline --no-backward --no-alpha0 --ag-leg 0 > $O/ncu_small.log 2>&1
