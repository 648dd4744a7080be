set -u
O=gpurun_out/r02n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_protocol.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in dlrm_small weak sweep_p1 sweep_p8; do
  timeout 600 python bench.py --config $c --no-cpu --no-alpha0 --ag-leg 0 --steps 30 --batches 8 --out $O/bench.jsonl > $O/bench_$c.log 2>&1
done
