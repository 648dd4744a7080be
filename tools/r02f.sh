set -u
O=gpurun_out/r02f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py --path ag_gemm --steps 20 --warmup 5 --out $O/ag_bench.jsonl > $O/ag_bench.log 2>&1; echo "rc=$?" >> $O/ag_bench.log
timeout 600 python bench.py --path ag_gemm --ag-config ag_small --steps 50 --warmup 5 --no-cpu --out $O/ag_bench.jsonl > $O/ag_bench_small.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ag_gemm_kernel -s 3 -c 1 -o $O/ag_full python bench.py --path ag_gemm --steps 3 --warmup 2 --no-cpu > $O/ncu_full.log 2>&1; echo "ncu rc=$?" >> $O/ncu_full.log
