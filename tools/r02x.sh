set -u
O=gpurun_out/r02x; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_bench_multirank.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --out $O/bench.jsonl > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
