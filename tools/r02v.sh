set -u
O=gpurun_out/r02v; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/bench_matrix.sh r02v > $O/matrix.log 2>&1
