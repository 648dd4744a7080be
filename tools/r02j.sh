set -u
O=gpurun_out/r02j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ag_gemm.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --path ag_gemm --steps 20 --warmup 5 --no-cpu --out $O/ag.jsonl > $O/ag.log 2>&1
timeout 600 python bench.py --path ag_gemm --ag-config ag_small --steps 50 --warmup 5 --no-cpu --out $O/ag.jsonl > $O/ag_small.log 2>&1
