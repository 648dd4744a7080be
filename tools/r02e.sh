set -u
O=gpurun_out/r02e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ag_gemm.py -x -q -k "fill or single_rank_exact" > $O/pytest1.log 2>&1; echo "rc=$?" >> $O/pytest1.log
timeout 900 python -m pytest tests/test_gpu_ag_gemm.py -q --durations=5 > $O/pytest2.log 2>&1; echo "rc=$?" >> $O/pytest2.log
