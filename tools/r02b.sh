set -u
O=gpurun_out/r02b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --out $O/bench.jsonl > $O/bench.log 2>&1
timeout 600 python bench.py --out-dtype bf16 --no-cpu --out $O/bench_bf16out.jsonl > $O/bench_bf16.log 2>&1
