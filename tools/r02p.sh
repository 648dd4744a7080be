set -u
O=gpurun_out/r02p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_backward.py tests/test_gpu_protocol.py -x -q --durations=8 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
