set -u
O=gpurun_out/r02c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/bench_matrix.sh r02c > $O/matrix.log 2>&1
bash tools/ncu_traffic.sh r02c > $O/ncu.log 2>&1
