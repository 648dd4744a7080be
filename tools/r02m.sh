set -u
O=gpurun_out/r02m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_smoke.py > $O/san_$t.log 2>&1; echo "rc=$?" >> $O/san_$t.log
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_smoke.py --W 2 > $O/san_memcheck_W2.log 2>&1; echo "rc=$?" >> $O/san_memcheck_W2.log
timeout 600 python bench.py --out $O/bench.jsonl > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 600 python bench.py --path ag_gemm --steps 20 --warmup 5 --out $O/ag.jsonl > $O/ag.log 2>&1; echo "rc=$?" >> $O/ag.log
