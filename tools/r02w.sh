set -u
O=gpurun_out/r02w2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ag_gemm.py tests/test_multiproc.py tests/test_bench_multirank.py -x -q -k "ag" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
