set -u
O=gpurun_out/r02aa2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_bench_multirank.py -q -k ablations > $O/pytest_abl.log 2>&1; echo "rc=$?" >> $O/pytest_abl.log
