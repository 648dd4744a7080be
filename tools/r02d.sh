set -u
O=gpurun_out/r02d; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --out $O/bench.jsonl > $O/bench.log 2>&1
